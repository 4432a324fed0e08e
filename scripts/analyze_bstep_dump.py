"""Dev aid: per-column b-step records (EPC_BSTEP_TAIL=1 EPC_BSTEP_DUMP=file)
-> how predictable the heavy columns are from their first two SQP step
norms, and list-schedule makespans of column orderings on the resident warps
(durations as measured, so occupancy effects are ignored)."""
import heapq
import math
import sys

import numpy as np


def read(path):
    out = []
    with open(path, "rb") as f:
        while True:
            t = np.fromfile(f, np.int64, 1)
            if t.size == 0:
                break
            n = int(t[0])
            ns = np.fromfile(f, np.uint32, n).astype(np.float64)
            sqp = np.fromfile(f, np.int32, n)
            qp = np.fromfile(f, np.int32, n)
            sn = np.fromfile(f, np.float32, 2 * n).reshape(n, 2).astype(np.float64)
            out.append((ns, sqp, qp, sn))
    return out


def makespan(dur, order, slots):
    h = [0.0] * slots
    for c in order:
        t = heapq.heappop(h)
        heapq.heappush(h, t + dur[c])
    return max(h)


def two_phase(dur, sqp, est, slots, k=2, eager=None):
    """phase 1: every column runs min(k, sqp) iterations in queue order; a
    column predicted heavy (est >= eager) continues at once, the others'
    remainders are queued heaviest-predicted first after phase 1."""
    per = dur / np.maximum(sqp, 1)
    h = [(0.0, i) for i in range(slots)]
    heapq.heapify(h)
    deferred = []
    for c in range(len(dur)):
        t, w = heapq.heappop(h)
        first = per[c] * min(k, sqp[c])
        rest = dur[c] - first
        if eager is not None and est[c] >= eager:
            heapq.heappush(h, (t + dur[c], w))
        else:
            heapq.heappush(h, (t + first, w))
            if rest > 0:
                deferred.append((-est[c], c, rest))
    deferred.sort()
    for _, c, rest in deferred:
        t, w = heapq.heappop(h)
        heapq.heappush(h, (t + rest, w))
    return max(t for t, _ in h)


def main(path, slots=1184, tol=1e-2, cap=20):
    recs = read(path)
    print(f"{len(recs)} launches")
    for it, (ns, sqp, qp, sn) in enumerate(recs):
        if it % 10 and it != len(recs) - 1:
            continue
        ms = ns * 1e-6
        s0, s1 = sn[:, 0], sn[:, 1]
        q = np.where((s0 > 0) & (sqp >= 2), s1 / np.maximum(s0, 1e-300), 0.0)
        with np.errstate(divide="ignore", invalid="ignore"):
            rem = np.where((q > 0) & (q < 1), np.ceil(np.log(np.maximum(tol * s0 / np.maximum(s1, 1e-300), 1e-300)) / np.log(q)), cap)
        est = np.where(sqp <= 2, sqp, np.minimum(2 + np.maximum(rem, 0), cap))
        heavy = ms > 1.0
        flag = est >= 12
        base = makespan(ms, range(len(ms)), slots)
        lpt = makespan(ms, np.argsort(-ms), slots)
        tp = two_phase(ms, sqp, est, slots)
        tpe = two_phase(ms, sqp, est, slots, eager=12)
        print(f"launch {it:3d}: cols {len(ms)} mean {ms.mean():.3f} ms, max {ms.max():.2f}, sum/slots "
              f"{ms.sum() / slots:.3f}; heavy(>1ms) {heavy.sum()}, sqp20 {(sqp >= cap).sum()}; "
              f"est>=12 recall {(flag & heavy).sum() / max(heavy.sum(), 1):.2f} precision "
              f"{(flag & heavy).sum() / max(flag.sum(), 1):.2f}; corr(est, sqp) "
              f"{np.corrcoef(est, sqp)[0, 1]:.2f}")
        print(f"    makespan: queue {base:.3f}  LPT(oracle) {lpt:.3f}  two-phase {tp:.3f}  "
              f"two-phase+eager {tpe:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:3]))
