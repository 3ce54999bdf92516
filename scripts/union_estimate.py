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
