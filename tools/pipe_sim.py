"""Tiny discrete-event model of one SM of the prefix kernel (for choosing the MMA issue order).

Tensor pipe: FIFO of MMA jobs in issue order (S = 512 cyc, PV = 512 cyc for 128x128x128).
Softmax job of a row tile: fixed part `o1` (TMEM load + max), MUFU part `W` cycles at full
rate (processor-shared among the softmax warpgroups running MUFU at the same time), fixed `o2`.
"""
import argparse


def simulate(order, ntiles=40, W=1024, o1=350, o2=150, lat=120, mma=512, emu=0.0, nwg=2):
    W = W * (1 - emu)
    t_tensor = 0.0
    s_done = {}     # (tile, j) -> time S done
    p_done = {}     # (tile, j) -> time P published
    # softmax warpgroups run their jobs in j order; MUFU processor sharing approximated by
    # iterating: each softmax job's MUFU phase is stretched by the overlap with the other one.
    # We do a fixed-point iteration on the schedule.
    soft = {}
    for it in range(60):
        t_tensor = 0.0
        issue_t = 0.0
        s_done.clear()
        for (kind, tile, j) in order(ntiles, nwg):
            dep = 0.0
            if kind == "PV":
                dep = p_done.get((tile, j), 1e18)
            issue_t = max(issue_t, dep + lat) + 20
            start = max(t_tensor, issue_t)
            t_tensor = start + mma
            if kind == "S":
                s_done[(tile, j)] = t_tensor
        # softmax schedule with processor sharing against the other wg's MUFU intervals
        new_p = {}
        intervals = {w: [] for w in range(nwg)}
        for w in range(nwg):
            t = 0.0
            for j in range(ntiles):
                t = max(t, s_done.get((w, j), 1e18) + lat) + o1
                m0 = t
                # stretch by overlap with other wgs' MUFU intervals from previous iteration
                rem = W
                while rem > 1e-6:
                    others = sum(1 for w2 in range(nwg) if w2 != w for (a, b) in soft.get(w2, []) if a <= t < b)
                    rate = 1.0 / (1 + others)
                    # advance in small steps
                    step = min(rem / rate, 32.0)
                    t += step
                    rem -= step * rate
                intervals[w].append((m0, t))
                t += o2
                new_p[(w, j)] = t
        soft = intervals
        p_done = new_p
    end = max(p_done.values())
    return end / ntiles


def order_current(n, nwg):
    yield ("S", 0, 0)
    yield ("S", 1, 0)
    for j in range(n):
        yield ("PV", 0, j)
        if j + 1 < n:
            yield ("S", 0, j + 1)
        yield ("PV", 1, j)
        if j + 1 < n:
            yield ("S", 1, j + 1)


def order_s_first(n, nwg):
    """Issue the next S of the other tile before this tile's PV (one tile ahead)."""
    yield ("S", 0, 0)
    yield ("S", 1, 0)
    for j in range(n):
        yield ("PV", 0, j)
        yield ("PV", 1, j)
        if j + 1 < n:
            yield ("S", 0, j + 1)
            yield ("S", 1, j + 1)


if __name__ == "__main__":
    for name, o in [("current", order_current), ("pv-pv-s-s", order_s_first)]:
        for emu in (0.0, 0.25, 0.5):
            print(name, "emu", emu, "cycles/tile %.0f" % simulate(o, emu=emu))
