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


if __name__ == "__main__":
    out = {}
    for name in sys.argv[1:] or ["C0", "C1", "C2"]:
        out[name] = count(scenes.CONFIGS[name]())
        print(name, out[name])
    path = os.path.join(ROOT, "profiles", "b_alg.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(out)
    json.dump(old, open(path, "w"), indent=1)
