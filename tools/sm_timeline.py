"""Per-SM timeline of one k_raycast launch from tools/timeline.py's per-ray arrays
(gpurun_out/timeline_<cfg>.npy: start us, end us, SM id per pixel; DTSDF_STATS build).

Prints, per SM, when its first warp started, when its last warp ended and its warp-busy fraction
(sum of its 8x4-pixel warp tiles' durations over span x the SM's peak resident warps), then the
active-warp curve of the whole GPU in 40 bins and the drain: the time from the first SM going idle
to the kernel's end."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(name="C1"):
    a = np.load(os.path.join(ROOT, "gpurun_out", f"timeline_{name}.npy"))
    H, W = a.shape[:2]
    t = lambda x: x[: H // 4 * 4, : W // 8 * 8].reshape(H // 4, 4, W // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 32)
    st, en, sm = t(a[..., 0]).min(1), t(a[..., 1]).max(1), t(a[..., 2])[:, 0].astype(int)
    span = en.max()
    print(f"{name}: span {span:.1f} us, {len(st)} warp tiles on {len(np.unique(sm))} SMs")
    print(f"{'sm':>4} {'first':>7} {'last':>7} {'warps':>6} {'busy':>6}")
    rows = []
    for s in np.unique(sm):
        m = sm == s
        ev = np.concatenate([np.stack([st[m], np.ones(m.sum())], 1), np.stack([en[m], -np.ones(m.sum())], 1)])
        ev = ev[np.argsort(ev[:, 0], kind="stable")]
        peak = np.cumsum(ev[:, 1]).max()
        busy = (en[m] - st[m]).sum() / (span * peak)
        rows.append((s, st[m].min(), en[m].max(), m.sum(), busy))
    for r in rows:
        print(f"{r[0]:4d} {r[1]:7.1f} {r[2]:7.1f} {r[3]:6d} {r[4]:6.3f}")
    last = np.array([r[2] for r in rows])
    print(f"SM last-warp end: min {last.min():.1f} p10 {np.quantile(last, .1):.1f} median {np.median(last):.1f} "
          f"max {last.max():.1f} us -> drain (first idle SM to end) {span - last.min():.1f} us")
    bins = np.linspace(0, span, 41)
    act = [int(((st <= b) & (en > b)).sum()) for b in bins[:-1]]
    print("active warps, 40 bins of", f"{span / 40:.1f} us:", act)
    print(f"mean busy {np.mean([r[4] for r in rows]):.3f}")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["C1"]:
        main(n)
