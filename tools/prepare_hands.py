"""Write the caller-side hand fixtures assets/prepared/<hand>.hand.npz.

Hand loading (URDF parsing, convex hulls of the collision parts, dependency
groups) is the reference's caller-side step (load_hand stays
with the caller).  This script runs THE REFERENCE'S OWN load_hand
(hand.cpp:124-273, convex_hull convex.cpp:139-359, dependency_groups
hand.cpp:374-411 — oracle/_ref, compiled from /root/reference) once per bundled
hand and stores the result in the flat lg_hand_desc layout plus the visual
meshes and link names, so the product, the bench and the tests consume exactly
the reference's hand model without any loader of their own.  Run it where
/root/reference exists (the fixtures are committed; the GPU box only reads
them).

    python tools/prepare_hands.py
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref_py as R  # noqa: E402

HANDS = ["four_finger", "two_finger", "allegro_like", "leap_like", "shadow_like"]


def main():
    out_dir = os.path.join(ROOT, "assets", "prepared")
    os.makedirs(out_dir, exist_ok=True)
    for name in HANDS:
        urdf = os.path.join(ROOT, "assets", "hands", f"{name}.urdf")
        arrays = R.load_hand_arrays(urdf)
        arrays["source_urdf"] = np.array(f"assets/hands/{name}.urdf")
        arrays["source_sha256"] = np.array(hashlib.sha256(open(urdf, "rb").read()).hexdigest())
        path = os.path.join(out_dir, f"{name}.hand.npz")
        np.savez_compressed(path, **arrays)
        print(f"{path}: {arrays['n_links']} links, {arrays['dof']} dof, "
              f"{len(arrays['part_link'])} parts, {arrays['n_groups']} groups, "
              f"{os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
