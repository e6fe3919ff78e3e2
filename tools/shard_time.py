"""Per-rank layer time of the Ulysses head split: one C2 layer (pool + mask +
carve, k=0.08, p=0) on H_local = 24 / G heads, for G = 1, 2, 4, 8 -- the compute a rank does
between its all-to-alls.  Run once with TCB_CARVE_NOSPLIT=1 and once without to see what the
condition-row split does when few heads are local.

  python tools/shard_time.py [--out gpurun_out/shard_time.json]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench_suite  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    a = ap.parse_args()
    recs = []
    for G in (1, 2, 4, 8):
        H = 24 // G
        L = bench_suite.Layer((33, 45, 80), 256, H, 0.08)
        L.mask()
        t_mask = bench_suite.timed(L.mask)
        t_carve = bench_suite.timed(L.carve)
        pairs = L.pairs()
        recs.append({"G": G, "heads_local": H, "mask_ms": round(t_mask, 4), "carve_ms": round(t_carve, 4),
                     "layer_ms": round(t_mask + t_carve, 4),
                     "carve_tflops": round(4 * 128 * 128 * 128 * pairs / (t_carve * 1e-3) / 1e12, 1),
                     "split": os.environ.get("TCB_CARVE_NOSPLIT", "0") in ("", "0")})
        print(json.dumps(recs[-1]), flush=True)
    if a.out:
        json.dump(recs, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
