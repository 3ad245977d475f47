"""GPU-vs-oracle comparison with the tolerances BASELINE.json's north_star states:
hit/miss agreement >= 99.9 % of pixels; on agreeing hits depth within 1e-4 m and normals within
1e-3 rad; colour bit-exact after u8 rounding on >= 99.9 %.  Reading R20/R22: a pixel whose
depth or normal misses its tolerance counts against the same 0.1 % budget as a hit/miss
disagreement.  The direction mask must agree on >= 99.9 % of agreeing hits (stricter than the
north star, useful for debugging)."""
from __future__ import annotations

import numpy as np

DEPTH_TOL = 1e-4  # m
NORMAL_TOL = 1e-3  # rad
BUDGET = 1e-3


def to_np(x):
    if x is None:
        return None
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def compare(gpu: dict, ora: dict, budget: float = BUDGET) -> dict:
    gd = to_np(gpu["depth"]).astype(np.float64).reshape(-1)
    od = np.asarray(ora["depth"], np.float64).reshape(-1)
    n = gd.size
    gh, oh = gd > 0, od > 0
    both = gh & oh
    gn = to_np(gpu["normal"]).reshape(-1, 3).astype(np.float64)
    on = np.asarray(ora["normal"]).reshape(-1, 3)
    gc = to_np(gpu["color"]).reshape(-1, 3)
    oc = np.asarray(ora["color"]).reshape(-1, 3)
    gm = to_np(gpu["mask"]).reshape(-1)
    om = np.asarray(ora["mask"]).reshape(-1)
    derr = np.abs(gd - od)
    cosang = np.clip((gn * on).sum(1) / np.maximum(np.linalg.norm(gn, axis=1) * np.linalg.norm(on, axis=1), 1e-30),
                     -1, 1)
    nerr = np.arccos(cosang)
    bad_geom = both & ((derr > DEPTH_TOL) | (nerr > NORMAL_TOL))
    disagree = gh != oh
    st = {
        "pixels": int(n), "hits_gpu": int(gh.sum()), "hits_oracle": int(oh.sum()),
        "hit_disagree": int(disagree.sum()), "geom_out_of_tol": int(bad_geom.sum()),
        "budget_used": float((disagree.sum() + bad_geom.sum()) / max(n, 1)),
        "depth_max_err": float(derr[both].max()) if both.any() else 0.0,
        "depth_p999_err": float(np.quantile(derr[both], 0.999)) if both.any() else 0.0,
        "normal_max_err": float(nerr[both].max()) if both.any() else 0.0,
        "color_exact": float((gc[both] == oc[both]).all(1).mean()) if both.any() else 1.0,
        "mask_equal": float((gm[both] == om[both]).mean()) if both.any() else 1.0,
        "miss_outputs_zero": bool((gd[~gh] == 0).all() and (gn[~gh] == 0).all() and (gc[~gh] == 0).all()
                                  and (gm[~gh] == 0).all()),
    }
    return st


def assert_parity(gpu: dict, ora: dict, budget: float = BUDGET, what: str = "") -> dict:
    st = compare(gpu, ora, budget)
    assert st["budget_used"] <= budget, (what, st)
    assert st["color_exact"] >= 0.999, (what, st)
    assert st["mask_equal"] >= 0.999, (what, st)
    assert st["miss_outputs_zero"], (what, st)
    return st
