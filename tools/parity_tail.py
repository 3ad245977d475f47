"""Classify every GPU pixel outside the north-star geometric tolerances (hit/miss disagreement,
|depth - oracle| > 1e-4 m, normal angle > 1e-3 rad) by re-evaluating the fp64 oracle along that
pixel's ray (oracle.OracleVolume.eval, the O3 sample F(x, r)).  Calls oracle/ and scenes/ only to
classify; the GPU outputs are the ones under test.

Classes (readings R20 / R22 in DESIGN.md §4):
  R20_multi_root    depth: the GPU's root lies in the oracle's lattice bracket [t_{k-1}, t_k] and the
                    oracle's F has several sign changes there (a fine 4001-point scan), so both are
                    roots of F in the first bracket; the oracle's bisection picks one by its
                    midpoint decisions
  R22_lattice_flip  depth or hit/miss: the two sides bracket different lattice intervals; the oracle's
                    own values at the GPU's bracket ends show why it rejected it, and the margin of
                    that decision is at fp32 resolution: |f| < 2e-6, S < 1e-5, or the decision changes
                    when the sample moves by 4 fp32 ulps of its coordinates (F jumps at a cell face or
                    mixes thin-plate directions whose weights turn on a sub-micrometre scale)
  R22_normal_at_gpu_root  normal only: the oracle's normal evaluated at the GPU's root position
                    agrees with the GPU's normal within 1e-3 rad -- the difference is the root position
                    (within the depth tolerance), on a normal field that turns fast there
  R22_normal_kink   normal only: the oracle's own normal turns by more than 1e-3 rad when the sample
                    moves by 4 fp32 ulps (an ill-conditioned mixture of directions or a weight kink)
  unexplained       none of the above (the count the verdict asks to drive to zero)

    python tools/parity_tail.py [--c2-views 20] [--rooms 16] [--plates 8] [--spheres 8]
        -> gpurun_out/parity_tail.jsonl (one line per pixel) and a summary line per scene
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import scenes  # noqa: E402
from scenes.configs import ROOM_K, THETA, plate_cluster, room_patches, room_pose  # noqa: E402

DEPTH_TOL, NORMAL_TOL = 1e-4, 1e-3


def F(ov, o, r, t):
    s = ov.eval(o + t * r, r)
    return s


def normal_of(s):
    N = (s["W"][:, None] * s["nt"]).sum(0)
    n = np.linalg.norm(N)
    return N / n if n > 0 else N


def sign_changes(ov, o, r, t0, t1, n=4001):
    ts = np.linspace(t0, t1, n)
    vals = []
    for t in ts:
        s = F(ov, o, r, t)
        vals.append(s["f"] if s["valid"] else np.nan)
    v = np.array(vals)
    neg = v <= 0  # valid, f <= 0
    pos = ~neg    # valid f > 0 or invalid (an invalid sample counts as positive, reading R21)
    down = int((pos[:-1] & neg[1:]).sum())
    up = int((neg[:-1] & pos[1:]).sum())
    return down, up


def classify(ov, delta, theta, o, r, L, dg, do, ng, no):
    tg, to = dg * L, do * L
    rec = {}
    if dg > 0 and do > 0 and abs(dg - do) <= DEPTH_TOL:
        # normal only.  (1) the oracle's normal evaluated at the GPU's own root position: if it
        # agrees with the GPU normal, the difference is the root position (itself within the depth
        # tolerance); (2) how far the oracle's normal turns when the sample moves by 4 fp32 ulps
        ang = lambda p, q: float(np.arccos(np.clip(np.dot(p, q) / max(np.linalg.norm(p) * np.linalg.norm(q), 1e-30),
                                                   -1, 1)))
        a = ang(ng, no)
        sg = F(ov, o, r, tg)
        at_gpu_root = ang(normal_of(sg), ng) if sg["valid"] else None
        x0 = o + to * r
        s0 = ov.eval(x0, r)
        n0 = normal_of(s0)
        eps = 4 * np.spacing(np.float32(np.abs(x0).max()))
        turn = 0.0
        for ax in range(3):
            for sgn in (-1, 1):
                xp = x0.copy()
                xp[ax] += sgn * eps
                s = ov.eval(xp, r)
                if s["valid"]:
                    turn = max(turn, ang(n0, normal_of(s)))
        rec.update(kind="normal", normal_err=a, depth_err=float(abs(dg - do)),
                   oracle_normal_at_gpu_root_vs_gpu=at_gpu_root, oracle_normal_turn_4ulp=turn,
                   regime=int(s0["regime"]), W=[float(x) for x in s0["W"]])
        if at_gpu_root is not None and at_gpu_root <= NORMAL_TOL:
            rec["class"] = "R22_normal_at_gpu_root"
        elif turn > NORMAL_TOL:
            rec["class"] = "R22_normal_kink"
        else:
            rec["class"] = "unexplained"
        return rec
    # depth or hit/miss: which lattice brackets?
    kg = int(np.ceil(tg / delta - 1e-9)) if dg > 0 else None
    ko = int(np.ceil(to / delta - 1e-9)) if do > 0 else None
    rec.update(kind="hit_miss" if (dg > 0) != (do > 0) else "depth", depth_gpu=float(dg), depth_oracle=float(do),
               k_gpu=kg, k_oracle=ko)
    if kg is not None and kg == ko:
        down, up = sign_changes(ov, o, r, (ko - 1) * delta, ko * delta)
        rec.update(sign_changes_down=down, sign_changes_up=up)
        rec["class"] = "R20_multi_root" if down >= 2 or up >= 1 else "unexplained"
        return rec
    # different brackets: why does the oracle not take the GPU's bracket (or the GPU the oracle's)?
    margins = []
    for k in [x for x in (kg, ko) if x is not None]:
        for kk in (k - 1, k):
            s = F(ov, o, r, kk * delta)
            margins.append({"k": kk, "valid": bool(s["valid"]), "f": float(s["f"]), "S": float(s["S"]),
                            "regime": int(s["regime"])})
    # is a lattice sample's crossing decision (valid or not, and f > 0 or f <= 0) decided at
    # the fp32 resolution of the GPU's sample position?  The oracle is re-evaluated at the sample
    # moved by +-4 fp32 ulps of its largest coordinate along each axis: a decision that changes
    # there is position-sensitive at fp32 resolution (reading R22)
    flips = []
    for m in margins:
        x = o + m["k"] * delta * r
        eps = 4 * np.spacing(np.float32(np.abs(x).max()))
        base = (m["valid"], m["valid"] and m["f"] > 0)  # the crossing decision: valid, and which side
        for a in range(3):
            for sg in (-1, 1):
                xp = x.copy()
                xp[a] += sg * eps
                s = ov.eval(xp, r)
                if (s["valid"], s["valid"] and s["f"] > 0) != base:
                    flips.append({"k": m["k"], "axis": a, "sign": sg, "eps_m": float(eps), "f": float(s["f"]),
                                  "valid": bool(s["valid"])})
                    break
            else:
                continue
            break
    # an invalid sample whose weights are zero only by a kink: some direction with a gradient has
    # its membership argument <n, v^D> within 1e-6 of cos(theta) (w_dir's zero) or <n, -r> within
    # 1e-6 of 0 (the back-face clamp), so fp32 and fp64 may disagree on S > 0
    kinks = []
    for m in margins:
        if m["valid"]:
            continue
        s = ov.eval(o + m["k"] * delta * r, r)
        for D in range(6):
            if not s["has_grad"][D]:
                continue
            n = s["nt"][D]
            c = float(np.dot(n, scenes.DIRECTION_VECTORS[D]))
            nr = float(-np.dot(n, r))
            if abs(c - np.cos(theta)) < 1e-6 or abs(nr) < 1e-6:
                kinks.append({"k": m["k"], "D": D, "n_dot_v_minus_cos_theta": c - float(np.cos(theta)), "n_dot_minus_r": nr})
    rec["lattice_samples"] = margins
    rec["position_sensitive"] = flips
    rec["weight_kinks"] = kinks
    tiny = [m for m in margins if (m["valid"] and abs(m["f"]) < 2e-6) or (0 < m["S"] < 1e-5)]
    rec["class"] = "R22_lattice_flip" if (tiny or flips or kinks) else "unexplained"
    return rec


def scenes_list(args):
    out = []
    c2 = scenes.c2_thin()
    for v in range(args.c2_views):
        out.append(("C2", v, c2.volume, c2.poses[v], c2.intrinsics))
    c1 = scenes.c1_room()
    out.append(("C1", 0, c1.volume, c1.poses[0], c1.intrinsics))
    K = scenes.Intrinsics(**ROOM_K)
    for kind, n in (("room", args.rooms), ("plates", args.plates), ("sphere", args.spheres)):
        for s in range(n):
            seed = {"room": 7, "plates": 8, "sphere": 9}[kind]
            rng = np.random.default_rng([seed, 100 + s])
            Kc = K
            if kind == "sphere":
                vol = scenes.sphere_volume(radius=rng.uniform(0.12, 0.28), voxel_size=0.01, truncation=0.04, theta=THETA)
                d = rng.normal(size=3)
                d /= np.linalg.norm(d)
                pose = scenes.look_at(d * rng.uniform(0.45, 0.9), rng.uniform(-0.05, 0.05, size=3))
                Kc = scenes.Intrinsics(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)
            elif kind == "room":
                pat, pose = room_patches(rng, n_boxes=20), room_pose(rng)
                vol = scenes.patch_fill_c(pat, voxel_size=0.01, truncation=0.04, theta=THETA)
            else:
                pat, pose = plate_cluster(rng)
                vol = scenes.patch_fill_c(pat, voxel_size=0.005, truncation=0.02, theta=THETA)
            out.append((f"{kind}[{seed},{100 + s}]", 0, vol, pose, Kc))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2-views", type=int, default=20)
    ap.add_argument("--rooms", type=int, default=16)
    ap.add_argument("--plates", type=int, default=8)
    ap.add_argument("--spheres", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_tail.jsonl"))
    args = ap.parse_args()
    from paper_2301_12796_b200 import Renderer
    R = Renderer(0)
    fh = open(args.out, "w")
    totals = {}
    last_vol = None
    for name, view, vol, pose, K in scenes_list(args):
        if vol is not last_vol:
            R.upload_volume(vol)
            ov = oracle.OracleVolume(vol)
            last_vol = vol
        g = {k: v[0].cpu().numpy() for k, v in R.render(np.asarray(pose)[None], K).items()}
        o = ov.render(pose, K)
        gd, od = g["depth"].astype(np.float64), o["depth"]
        gn, on = g["normal"].astype(np.float64), o["normal"]
        both = (gd > 0) & (od > 0)
        cosang = np.clip((gn * on).sum(-1) / np.maximum(np.linalg.norm(gn, axis=-1) * np.linalg.norm(on, axis=-1),
                                                        1e-30), -1, 1)
        bad = ((gd > 0) != (od > 0)) | (both & ((np.abs(gd - od) > DEPTH_TOL) | (np.arccos(cosang) > NORMAL_TOL)))
        vv, uu = np.nonzero(bad)
        counts = {}
        for u, v in zip(uu, vv):
            oo, r, L = oracle.ray_dirs(pose, K, np.array([[u, v]], np.int32))
            # the oracle's own lattice step and theta: the float32 values the C ABI receives
            rec = classify(ov, float(np.float32(vol.delta)), float(np.float32(vol.theta)), oo, r[0], float(L[0]),
                           float(gd[v, u]), float(od[v, u]), gn[v, u], on[v, u])
            rec.update(scene=name, view=view, pixel=[int(u), int(v)], normal_gpu=[float(x) for x in gn[v, u]],
                       normal_oracle=[float(x) for x in on[v, u]])
            fh.write(json.dumps(rec) + "\n")
            counts[rec["class"]] = counts.get(rec["class"], 0) + 1
            totals[rec["class"]] = totals.get(rec["class"], 0) + 1
        line = {"scene": name, "view": view, "pixels": int(gd.size), "out_of_tolerance": int(bad.sum()), "classes": counts}
        print(json.dumps(line), flush=True)
        fh.write(json.dumps(line) + "\n")
    print(json.dumps({"summary": totals}), flush=True)
    fh.write(json.dumps({"summary": totals}) + "\n")


if __name__ == "__main__":
    main()
