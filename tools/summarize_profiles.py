"""Summarise a tools/profile_round.sh bundle (gpurun_out/<tag>_*) into profiles/ (tracked).

    python tools/summarize_profiles.py TAG [WORKLOAD]

Writes profiles/<tag>_summary.md (bench line, clocks, launch-list shares, the key ncu --set full
counters of the prefix and tree/merge kernels), copies the bench JSON and the launch CSV, and
updates profiles/traffic_<workload>.json (dram bytes per launch of the prefix kernel, which
bench.py reports as roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import shutil
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.max", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return None, []
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        launches.append({h: (u, v) for h, u, v in zip(hdr, units, r)})
    return hdr, launches


def to_bytes(unit, val):
    v = float(val.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    tag = sys.argv[1]
    workload = sys.argv[2] if len(sys.argv) > 2 else "llama8b_64k"
    os.makedirs(PROF, exist_ok=True)
    md = [f"# Profile bundle `{tag}` (tools/profile_round.sh on one B200; summarised by tools/summarize_profiles.py)", ""]
    bj = os.path.join(OUT, f"{tag}_bench.json")
    if os.path.exists(bj):
        shutil.copy(bj, os.path.join(PROF, f"{tag}_bench.json"))
        line = json.loads(open(bj).read().strip().splitlines()[-1])
        r = line.get("roofline") or {}
        md += ["## Bench line (`python bench.py`, default workload)", "",
               f"- value {line['value']:.4g} {line['unit']}, {line['us_per_step']:.1f} µs/step; "
               f"e2e {line['e2e']['value']:.4g} {line['e2e']['unit']}",
               f"- prefix kernel {r.get('kernel_us', 0):.1f} µs (CUDA events, live); roofline "
               f"{r.get('roofline_us', 0):.1f} µs ({r.get('bound')}); frac {r.get('frac', 0):.3f} of measured; "
               f"{r.get('hbm_gbs_achieved', 0):.0f} GB/s, {r.get('tflops_achieved', 0):.0f} TFLOP/s",
               f"- clocks {line.get('clocks')}", ""]
        if "all_configs_us_per_step" in line:
            md += ["| workload | µs/step | prefix µs | roofline µs | prefix frac | tokens/s |", "|---|---|---|---|---|---|"]
            for k, v in line["all_configs_us_per_step"].items():
                md.append(f"| {k} | {v['us_per_step']:.1f} | {v['prefix_us']:.1f} | {v['roofline_us']:.1f} | "
                          f"{v['prefix_frac_of_roofline']:.3f} | {v['tokens_per_s']:.4g} |")
            md.append("")
    lc = os.path.join(OUT, f"{tag}_launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(PROF, f"{tag}_launches.csv"))
        rows = [r for r in csv.reader(open(lc)) if len(r) > 10]
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        d = collections.defaultdict(list)
        for r in rows[1:]:
            d[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
        ours = {k: v for k, v in d.items() if "hta::" in k}
        tot = sum(statistics.mean(v) for v in ours.values())
        md += ["## Launch list (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised)", "",
               "| kernel | launches | mean µs | share of our step |", "|---|---|---|---|"]
        for k, v in sorted(d.items(), key=lambda kv: -statistics.mean(kv[1])):
            share = f"{statistics.mean(v) / tot:.1%}" if k in ours else "(not ours: L2 flush)"
            md.append(f"| `{k}` | {len(v)} | {statistics.mean(v) / 1e3:.2f} | {share} |")
        md.append("")
    for kern, rep in (("prefix_tc_kernel", f"{tag}_prefix.ncu-rep"), ("tree_merge_kernel", f"{tag}_treemerge.ncu-rep")):
        path = os.path.join(OUT, rep)
        if not os.path.exists(path):
            continue
        hdr, launches = ncu_raw(path)
        if not launches:
            continue
        L = launches[-1]
        md += [f"## `{kern}` — ncu --set full (one launch)", "", "| counter | value |", "|---|---|"]
        for k in KEYS:
            if k in L:
                md.append(f"| {k} | {L[k][1]} {L[k][0]} |")
        md.append("")
        if kern == "prefix_tc_kernel":
            rb = to_bytes(*L["dram__bytes_read.sum"])
            wb = to_bytes(*L["dram__bytes_write.sum"])
            json.dump({"tag": tag, "kernel": kern, "dram_bytes_read": rb, "dram_bytes_write": wb,
                       "dram_bytes_per_launch": rb + wb, "source": f"profiles/{tag}_summary.md"},
                      open(os.path.join(PROF, f"traffic_{workload}.json"), "w"), indent=1)
    ck = os.path.join(OUT, f"{tag}_clocks.csv")
    if os.path.exists(ck):
        sm, reasons = [], set()
        for r in list(csv.reader(open(ck)))[1:]:
            try:
                sm.append(float(r[1].split()[0]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal", "sw_thermal", "sw_power_cap"), r[5:9]):
                if "Active" in v and "Not" not in v:
                    reasons.add(name)
        if sm:
            md += ["## Clocks during the bench (nvidia-smi -lms 200)", "",
                   f"{len(sm)} samples, SM MHz median {statistics.median(sm):.0f}, min {min(sm):.0f}, "
                   f"max {max(sm):.0f}; reasons active: {sorted(reasons) or 'none'}", ""]
    open(os.path.join(PROF, f"{tag}_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
