"""Issued 128x128 key tiles per head for one call, 128-row-aligned query tiles
vs block-aligned ones (two 64-row blocks per tile), from the oracle's
selection on the bench's synthetic inputs (CPU; dev tool, not a test).

    I=14 S=0.9046 python scripts/union_estimate.py     # c3
    I=7 S=0.5 python scripts/union_estimate.py         # c5_s50
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lf_oracle as O  # noqa: E402

f, n, b = 3, 1560, 64
i = int(os.environ.get("I", "14"))
s = float(os.environ.get("S", "0.904632706980882"))
lq, lk, d = f * n, i * f * n, 128
q, k, v = O.synthetic_qkv(1, lq, lk, d, heads=1)
views, sel = O.select(q[0], k[0], i, s, f, n, b, b, 6, "global", framewise=True)
qt = O.q_tiling(f, n, b, True)
P = (i - 1) * f * views.blocks_per_frame
past = sel.bits[:, :P]
nqb = past.shape[0]


def issued(tiles):
    t = 0
    for blks in tiles:
        u = np.zeros(P, bool)
        for r in blks:
            u |= past[r]
        t += -(-int(u.sum()) // 2)  # 64-key segments, two per 128-key tile
    return t


def block_of(row):
    tt = row // n
    return tt * qt.per_period + (row - tt * n) // b


aligned = [list(range(block_of(q0), block_of(min(q0 + 128, lq) - 1) + 1)) for q0 in range(0, lq, 128)]
blockwise = []
for fr in range(f):
    bl = list(range(fr * qt.per_period, (fr + 1) * qt.per_period))
    blockwise += [bl[j:j + 2] for j in range(0, len(bl), 2)]
kt_cur = -(-lq // 128)
eff = sum(int(past[r].sum()) for r in range(nqb)) * 64 * 64 / (128 * 128) + lq * lq / (128 * 128)
a = issued(aligned) + len(aligned) * kt_cur
bw = issued(blockwise) + len(blockwise) * kt_cur
print(f"chunk {i}, s={s}: selected past blocks per query block {past.sum() / nqb:.1f}")
print(f"effective tile-equivalents {eff:.0f}")
print(f"128-row tiles: {len(aligned)} query tiles, issued {a} (eff/issued {eff / a:.2f})")
print(f"block-aligned: {len(blockwise)} query tiles, issued {bw} (eff/issued {eff / bw:.2f}), "
      f"{100 * (bw - a) / a:+.1f} %")

# greedy pairing of query blocks by selection overlap (largest shared 64-key
# segment count first), within the head; unpaired blocks ride alone
def overlap_pairs():
    sets = [past[r] for r in range(nqb)]
    left = set(range(nqb))
    pairs = []
    cand = []
    for a_ in range(nqb):
        for b_ in range(a_ + 1, nqb):
            cand.append((int((sets[a_] & sets[b_]).sum()), a_, b_))
    cand.sort(reverse=True)
    for ov, a_, b_ in cand:
        if a_ in left and b_ in left:
            pairs.append([a_, b_])
            left.discard(a_)
            left.discard(b_)
    pairs += [[r] for r in sorted(left)]
    return pairs


jp = overlap_pairs()
jw = issued(jp) + len(jp) * kt_cur
print(f"overlap-paired: {len(jp)} query tiles, issued {jw} (eff/issued {eff / jw:.2f}), "
      f"{100 * (jw - a) / a:+.1f} % vs 128-row, {100 * (jw - bw) / bw:+.1f} % vs block-aligned")


# pairing by sorting query blocks on their retrieved-frame set (the kernel's
# cheap surrogate for overlap pairing): equal frame sets end up adjacent
def frame_sort_pairs():
    keys = []
    for r in range(nqb):
        fr = sorted(int(t) for t in sel.frames[r] if t < (i - 1) * f)
        keys.append((tuple(fr), r))
    order = [r for _, r in sorted(keys)]
    return [order[j:j + 2] for j in range(0, len(order), 2)]


fp = frame_sort_pairs()
fw_ = issued(fp) + len(fp) * kt_cur
print(f"frame-sorted:   {len(fp)} query tiles, issued {fw_} (eff/issued {eff / fw_:.2f}), "
      f"{100 * (fw_ - bw) / bw:+.1f} % vs block-aligned")


def mutual_best_pairs(max_rounds):
    """The device kernel's mutual-best rounds (pairing.cuh), at most max_rounds."""
    ov = np.zeros((nqb, nqb), np.int64)
    for a_ in range(nqb):
        for b_ in range(nqb):
            if a_ != b_:
                ov[a_, b_] = int((past[a_] & past[b_]).sum())
    mate = [-1] * nqb
    rounds = 0
    for _ in range(max_rounds):
        prop = []
        for x in range(nqb):
            best, key = -1, None
            if mate[x] < 0:
                for y in range(nqb):
                    if y == x or mate[y] >= 0:
                        continue
                    k2 = (ov[x, y], -abs(x - y), -y)
                    if key is None or k2 > key:
                        key, best = k2, y
            prop.append(best)
        new = 0
        for x in range(nqb):
            y = prop[x]
            if y >= 0 and prop[y] == x:
                mate[x] = y
                new += 1
        rounds += 1
        if new == 0:
            break
    pairs, pend = [], None
    for x in range(nqb):
        y = mate[x]
        if y >= 0:
            if x < y:
                pairs.append([x, y])
        elif pend is None:
            pend = x
        else:
            pairs.append([pend, x])
            pend = None
    if pend is not None:
        pairs.append([pend])
    return pairs, rounds


for R in (2, 4, 8, 100):
    mp, rr = mutual_best_pairs(R)
    mw = issued(mp) + len(mp) * kt_cur
    print(f"mutual-best <= {R} rounds (ran {rr}): issued {mw}, {100 * (mw - bw) / bw:+.1f} % vs block-aligned")
