/*
 * hta_oracle.c -- TEST INFRASTRUCTURE ONLY (never linked into, or called by, the product).
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of the attention that
 * LongSpec's Hybrid Tree Attention computes (arXiv 2502.17421).  It shares no code,
 * header, table or helper with the CUDA library; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * What it computes ("Splitting Key-Value Pairs"; Appendix C,
 * PAPER.md:603-656):  for every batch b, tree token t and query head h,
 *
 *     o = softmax( q K_merge^T / sqrt(d) ) V_merge
 *
 * where K_merge = [K_cache ; K_specs] and the row's visibility is the EXPLICIT mask row
 * [ 1 ... 1 (cache part, "do not require additional masks") |
 *   tree-mask row (specs part, "need masking") ].
 * LSE = log sum_j exp(Z_j)  (natural log of the scaled logits).
 *
 * Algorithm, in the order of SURVEY.md §8(c) O1-O7 (no blocking, no online softmax):
 *   O1  g = h / (H / H_kv)  (grouped-query heads share KV head g; reading Z8);
 *       n = cache_seqlens[b].
 *   O2  build the explicit mask row m[0 .. n+T): m[j] = 1 for visible cache columns
 *       j < n (restricted to [cache_lo, cache_hi) when a sub-range is requested), and
 *       m[n+s] = mask[b][t][s] for the tree part.
 *   O3  z_j = scale * sum_k q[k] * K_j[k]  in double for every j with m[j] = 1.
 *   O4  mx = max_j z_j; if no column is visible: O = 0, LSE = -inf (sentinel, Z10).
 *   O5  w_j = exp(z_j - mx); s = sum_j w_j (sequential in j); LSE = mx + log(s).
 *   O6  O[k] = (sum_j w_j V_j[k]) / s.
 *   O7  partials: the same with only cache columns (part=1) or only tree columns (part=2).
 *
 * Inputs are float32 arrays holding the exact values the GPU consumes (bf16 values are
 * exactly representable in float32); every product and sum is in double.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int B, T, H, Hkv, d;
    long N;                 /* cache capacity (sequence extent of kc/vc) */
    double scale;
    const float *q;         /* [B, T, H, d]     */
    const float *kc, *vc;   /* [B, N, Hkv, d]   */
    const int32_t *seqlens; /* [B] (NULL: all N) */
    const float *kt, *vt;   /* [B, T, Hkv, d]   */
    const uint8_t *mask;    /* [B, T, T]        */
    int part;               /* 0: cache + tree, 1: cache only, 2: tree only */
    long cache_lo, cache_hi;/* visible cache sub-range (clipped to [0, n)) */
    /* rows to compute: (b, t, h) triples; NULL = all rows in [B, T, H] order */
    const int32_t *rows;
    long n_rows;
    double *o;              /* [n_rows, d] */
    double *lse;            /* [n_rows]    */
    /* thread bookkeeping */
    long next_row;
    pthread_mutex_t lock;
} oracle_job;

static void row_coords(const oracle_job *J, long r, int *b, int *t, int *h) {
    if (J->rows) {
        *b = J->rows[3 * r + 0];
        *t = J->rows[3 * r + 1];
        *h = J->rows[3 * r + 2];
    } else {
        *h = (int)(r % J->H);
        *t = (int)((r / J->H) % J->T);
        *b = (int)(r / ((long)J->H * J->T));
    }
}

/* One output row, steps O1-O6. */
static void oracle_row(const oracle_job *J, long r, uint8_t *mrow, double *z, double *acc) {
    int b, t, h;
    row_coords(J, r, &b, &t, &h);
    const int d = J->d, T = J->T;
    const int G = J->H / J->Hkv;
    const int g = h / G;                                              /* O1 */
    const long n = J->seqlens ? (long)J->seqlens[b] : J->N;
    const long ncol = n + T;

    /* O2: explicit mask row over [cache | tree] */
    for (long j = 0; j < n; ++j)
        mrow[j] = (J->part != 2 && j >= J->cache_lo && j < J->cache_hi) ? 1 : 0;
    for (int s = 0; s < T; ++s)
        mrow[n + s] = (J->part != 1) ? J->mask[((long)b * T + t) * T + s] : 0;

    const float *qv = J->q + (((long)b * T + t) * J->H + h) * d;

    /* O3: logits in double */
    double mx = -INFINITY;
    int any = 0;
    for (long j = 0; j < ncol; ++j) {
        if (!mrow[j]) continue;
        const float *kv = (j < n) ? J->kc + (((long)b * J->N + j) * J->Hkv + g) * d
                                  : J->kt + (((long)b * T + (j - n)) * J->Hkv + g) * d;
        double dot = 0.0;
        for (int k = 0; k < d; ++k) dot += (double)qv[k] * (double)kv[k];
        z[j] = J->scale * dot;
        if (!any || z[j] > mx) mx = z[j];                             /* O4 */
        any = 1;
    }
    double *o = J->o + r * d;
    if (!any) {                                                       /* O4 sentinel */
        for (int k = 0; k < d; ++k) o[k] = 0.0;
        J->lse[r] = -INFINITY;
        return;
    }
    /* O5 + O6 */
    double s = 0.0;
    for (int k = 0; k < d; ++k) acc[k] = 0.0;
    for (long j = 0; j < ncol; ++j) {
        if (!mrow[j]) continue;
        const double w = exp(z[j] - mx);
        s += w;
        const float *vv = (j < n) ? J->vc + (((long)b * J->N + j) * J->Hkv + g) * d
                                  : J->vt + (((long)b * T + (j - n)) * J->Hkv + g) * d;
        for (int k = 0; k < d; ++k) acc[k] += w * (double)vv[k];
    }
    J->lse[r] = mx + log(s);
    for (int k = 0; k < d; ++k) o[k] = acc[k] / s;
}

static void *oracle_worker(void *arg) {
    oracle_job *J = (oracle_job *)arg;
    const long ncol_max = J->N + J->T;
    uint8_t *mrow = (uint8_t *)malloc((size_t)ncol_max + 1);
    double *z = (double *)malloc(sizeof(double) * ((size_t)ncol_max + 1));
    double *acc = (double *)malloc(sizeof(double) * (size_t)J->d);
    for (;;) {
        pthread_mutex_lock(&J->lock);
        long r = J->next_row++;
        pthread_mutex_unlock(&J->lock);
        if (r >= J->n_rows) break;
        oracle_row(J, r, mrow, z, acc);
    }
    free(mrow);
    free(z);
    free(acc);
    return NULL;
}

/* Returns 0 on success, -1 on bad arguments. */
int oracle_attention(int B, int T, int H, int Hkv, int d, long N, double scale,
                     const float *q, const float *kc, const float *vc, const int32_t *seqlens,
                     const float *kt, const float *vt, const uint8_t *mask,
                     int part, long cache_lo, long cache_hi,
                     const int32_t *rows, long n_rows,
                     double *o, double *lse, int nthreads) {
    if (B < 0 || T < 0 || H <= 0 || Hkv <= 0 || d <= 0 || N < 0 || H % Hkv) return -1;
    if (seqlens)
        for (int b = 0; b < B; ++b)
            if (seqlens[b] < 0 || seqlens[b] > N) return -1;
    oracle_job J;
    memset(&J, 0, sizeof(J));
    J.B = B; J.T = T; J.H = H; J.Hkv = Hkv; J.d = d; J.N = N; J.scale = scale;
    J.q = q; J.kc = kc; J.vc = vc; J.seqlens = seqlens; J.kt = kt; J.vt = vt; J.mask = mask;
    J.part = part; J.cache_lo = cache_lo; J.cache_hi = cache_hi;
    J.rows = rows;
    J.n_rows = rows ? n_rows : (long)B * T * H;
    J.o = o; J.lse = lse;
    J.next_row = 0;
    pthread_mutex_init(&J.lock, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, oracle_worker, &J);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    pthread_mutex_destroy(&J.lock);
    return 0;
}
