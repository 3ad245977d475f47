"""Algorithmic bytes per ray counted by the instrumented CPU oracle.

    b_alg = 20 B (outputs) + (U_vox * 8 B + U_rgb * 3 B + U_idx * 32 B) / rays

U_vox: distinct (voxel, direction) {sdf f32, weight f32} records read by any sample evaluation
of any ray of the view; U_rgb: distinct colour records read by shading; U_idx: distinct
allocated block locations resolved (one 32-B hash entry each).  Calls only oracle/ and scenes/;
writes profiles/b_alg.json.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import scenes  # noqa: E402


def count(w, view=0):
    ov = oracle.OracleVolume(w.volume, counting=True)
    K = w.intrinsics
    ov.render(w.poses[view], K)
    c = ov.counts()
    rays = K.width * K.height
    b = 20.0 + (c["voxel_records"] * 8 + c["rgb_records"] * 3 + c["locations"] * 32) / rays
    return {"bytes_per_ray": b, "rays": rays, "U_vox": c["voxel_records"], "U_rgb": c["rgb_records"],
            "U_idx": c["locations"], "view": view,
            "formula": "20 + (U_vox*8 + U_rgb*3 + U_idx*32) / rays"}


def count_batch(w, n_views=256):
    """configs[3]: the union of the records any ray of any of the batch's views reads (one counting
    volume across the views), over all the batch's rays -- the algorithmic bytes of one batch."""
    ov = oracle.OracleVolume(w.volume, counting=True)
    K = w.intrinsics
    for v in range(n_views):
        ov.render(w.poses[v], K)
    c = ov.counts()
    rays = K.width * K.height * n_views
    b = 20.0 + (c["voxel_records"] * 8 + c["rgb_records"] * 3 + c["locations"] * 32) / rays
    return {"bytes_per_ray": b, "rays": rays, "U_vox": c["voxel_records"], "U_rgb": c["rgb_records"],
            "U_idx": c["locations"], "views": n_views,
            "formula": "20 + (U_vox*8 + U_rgb*3 + U_idx*32) / rays, U over the union of the batch's views"}


def count_tiles(w, views=(0, 16, 32, 48), tile=(80, 60)):
    """configs[4]: the brute-force oracle march over 5 mm voxels is too slow for whole frames, so
    the counts come from contiguous pixel tiles (80 x 60, 1/64 of a frame) at the centres of the
    four image quadrants of 4 of the 64 views, each tile counted with its own counting volume (so
    neighbouring rays share records as in a full frame; tile borders slightly overstate b_alg)."""
    K = w.intrinsics
    tot = {"voxel_records": 0, "rgb_records": 0, "locations": 0}
    rays = 0
    for v in views:
        for qx in (0, 1):
            for qy in (0, 1):
                u0 = K.width // 4 + qx * K.width // 2 - tile[0] // 2
                v0 = K.height // 4 + qy * K.height // 2 - tile[1] // 2
                vv, uu = [a.ravel() for a in np.mgrid[v0:v0 + tile[1], u0:u0 + tile[0]]]
                px = np.stack([uu, vv], 1).astype(np.int32)
                ov = oracle.OracleVolume(w.volume, counting=True)
                ov.render(w.poses[v], K, pixels=px)
                c = ov.counts()
                for k in tot:
                    tot[k] += c[k]
                rays += len(px)
                del ov
    b = 20.0 + (tot["voxel_records"] * 8 + tot["rgb_records"] * 3 + tot["locations"] * 32) / rays
    return {"bytes_per_ray": b, "rays": rays, "U_vox": tot["voxel_records"], "U_rgb": tot["rgb_records"],
            "U_idx": tot["locations"], "views": list(views), "tiles": "80x60 at the 4 quadrant centres per view",
            "formula": "20 + (sum U_vox*8 + sum U_rgb*3 + sum U_idx*32) / rays over the tiles"}


if __name__ == "__main__":
    import numpy as np  # noqa: F401
    out = {}
    for name in sys.argv[1:] or ["C0", "C1", "C2"]:
        if name == "C3":
            out[name] = count_batch(scenes.CONFIGS[name]())
        elif name == "C4":
            out[name] = count_tiles(scenes.CONFIGS[name]())
        else:
            out[name] = count(scenes.CONFIGS[name]())
        print(name, out[name], flush=True)
    path = os.path.join(ROOT, "profiles", "b_alg.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(out)
    json.dump(old, open(path, "w"), indent=1)
