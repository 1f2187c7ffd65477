"""Summarises an RF_TRACE_FILE timeline (per-pass u64 records written by the
tracking kernel): for each pass, lead-CTA start, lead tiles done, slowest CTA
tiles done, all-reduce done; the gap to the next pass start is the LM solve."""
import sys
from collections import defaultdict

import numpy as np


def main(path, skip=3):
    raw = np.fromfile(path, dtype=np.uint64).reshape(-1, 256, 8)[skip:]
    per = defaultdict(list)
    verdicts = defaultdict(lambda: [0, 0, 0])
    frame_tot = []
    mask = raw[:, 255, :7].astype(np.float64)
    mask = mask[mask[:, 0] > 0]
    if len(mask):
        d = np.diff(mask, axis=1) / 1e3
        print("mask stages (us): threshold %.1f  erode %.1f  stamp-init %.1f  floodfill %.1f  dilate %.1f  count %.1f"
              % tuple(d.mean(0)))
    ff = raw[:, 254, :2].astype(np.float64)
    ff = ff[ff[:, 0] > 0]
    if len(ff):
        print("floodfill per frame: seeded tiles %.1f, sweeps %.1f" % tuple(ff.mean(0)))
    rs = raw[:, 253, :8].astype(np.float64)  # floodfill round starts (CTA 0)
    rd = raw[:, 252, :8].astype(np.float64)  # slowest CTA's tiles done per round
    if (rs[:, 0] > 0).any():
        tiles, bar = [], []
        for a, b in zip(rs, rd):
            n = int((a > 0).sum())
            for r in range(n):
                tiles.append((b[r] - a[r]) / 1e3)
                if r + 1 < n:
                    bar.append((a[r + 1] - b[r]) / 1e3)
        print("floodfill rounds: tiles (slowest) %.2f us, barrier+next %.2f us per round" % (np.mean(tiles), np.mean(bar) if bar else 0))
    for fr in raw:
        fr = fr[:252]
        passes = fr[fr[:, 0] > 0]
        if len(passes) == 0:
            continue
        frame_tot.append((int(passes[-1, 3]) - int(passes[0, 0])) / 1e3)
        for i, p in enumerate(passes):
            start, lead_done, slow_done, red_done, level, px, jac, _ = (int(x) for x in p[:8])
            nxt = int(passes[i + 1, 0]) if i + 1 < len(passes) else red_done
            solved = int(passes[i + 1, 7]) if i + 1 < len(passes) and int(passes[i + 1, 7]) > red_done else 0
            verdict = jac >> 8  # 1 accepted, 2 rejected, 0 not a trial (first pass of a level)
            jac &= 0xFF
            verdicts[(level, px, jac)][verdict] += 1
            key = (level, px, jac)
            per[key].append((slow_done - start, red_done - slow_done, max(0, nxt - red_done), lead_done - start,
                             (solved - red_done) if solved else np.nan, (nxt - solved) if solved else np.nan))
    print(f"frames {len(frame_tot)}  mean tracked span {np.mean(frame_tot):.1f} us")
    print("level    px  jac  passes/frame  tiles(slowest)  reduce+release  gap  lead-tiles  "
          "[gap = solve-done + sync]  (us)")
    for key in sorted(per):
        a = np.array(per[key]) / 1e3
        print(f"{key[0]:5d} {key[1]:7d} {key[2]:3d} {len(a) / len(frame_tot):10.1f} "
              f"{a[:, 0].mean():14.2f} {a[:, 1].mean():14.2f} {a[:, 2].mean():6.2f} {a[:, 3].mean():10.2f}  "
              f"[{np.nanmean(a[:, 4]):.2f} + {np.nanmean(a[:, 5]):.2f}]  "
              f"trials accepted/rejected per frame {verdicts[key][1] / len(frame_tot):.1f}/{verdicts[key][2] / len(frame_tot):.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
