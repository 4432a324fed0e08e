"""Dev aid: list-schedule simulation of b-step claim orders on per-column
records of consecutive launches (EPC_BSTEP_TAIL=1 EPC_BSTEP_DUMP=file
EPC_BSTEP_DUMP_EVERY=1): the queue's natural order, longest-first on the
previous launch's costs, longest-first on the launch's own costs (an oracle),
and how many columns' cost more than doubled to over 1 ms ("jumpers")."""
import heapq
import sys

import numpy as np

from analyze_bstep_dump import read


def sim(dur, order, slots):
    h = [0.0] * slots
    for c in order:
        heapq.heappush(h, heapq.heappop(h) + dur[c])
    return max(h)


def main(path, slots=1184):
    recs = read(path)
    for t in range(2, len(recs)):
        prev, cur = recs[t - 1][0] * 1e-6, recs[t][0] * 1e-6
        sq_prev = recs[t - 1][1]
        n = len(cur)
        j = (cur > 1.0) & (cur > 2 * prev)
        print(f"launch {t}: ideal {cur.sum() / slots:.2f} ms, natural {sim(cur, range(n), slots):.2f}, "
              f"longest-first on previous costs {sim(cur, np.argsort(-prev, kind='stable'), slots):.2f}, "
              f"on own costs {sim(cur, np.argsort(-cur), slots):.2f}; jumpers {int(j.sum())} "
              f"(median previous SQP count {int(np.median(sq_prev[j])) if j.any() else 0})")


if __name__ == "__main__":
    main(sys.argv[1])
