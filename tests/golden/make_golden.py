"""Generate the golden k-NN fixtures from the UNMODIFIED reference library.

Run in the build container (needs oracle/_ref/libtknn_ref_capi.so, i.e. the
reference compiled from /root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Each case stores only the small outputs (neighbor indices and distance bits)
plus the recipe for its inputs (generator + seed, or explicit values); the
inputs are regenerated at test time with the C restatement's SplitMix64,
whose bit-equality with the reference generator is itself pinned by
tests/test_oracle_pin.py.  Everything lands in golden.npz.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import METRICS, Reference, normalize_rows  # noqa: E402

# (name, n, d, k, metric, seed, transform)
CASES = [
    ("hel_300x17_k12", 300, 17, 12, "hellinger", 5, None),
    ("sq_300x17_k12", 300, 17, 12, "sqeuclidean", 5, None),
    ("cos_300x17_k12", 300, 17, 12, "cosine", 5, "normalize"),
    ("sq_1000x64_k10", 1000, 64, 10, "sqeuclidean", 42, None),
    ("sq_400x33_k100", 400, 33, 100, "sqeuclidean", 7, None),
    ("hel_513x129_k32", 513, 129, 32, "hellinger", 11, None),
    ("sq_2048x256_k10", 2048, 256, 10, "sqeuclidean", 1, None),
    ("sq_ties_400x3_k20", 400, 3, 20, "sqeuclidean", 3, "quantize"),
    ("sq_k_full_40x5", 40, 5, 1000, "sqeuclidean", 9, None),
    ("cos_1024x128_k32", 1024, 128, 32, "cosine", 3, "normalize"),
]


def make_input(gen, n, d, seed, transform):
    x = gen(n, d, seed)
    if transform == "normalize":
        x = normalize_rows(x)
    elif transform == "quantize":
        # Coarse grid -> many exactly tied distances; exercises the index
        # tie-break of the (distance, index) order (heap.hpp:21-24).
        x = np.floor(x * 4.0).astype(np.float32)
    return np.ascontiguousarray(x, dtype=np.float32)


def main():
    ref = Reference()
    out = {}
    meta = []
    for name, n, d, k, metric, seed, transform in CASES:
        x = make_input(ref.generate, n, d, seed, transform)
        idx, dist, pairs, _ = ref.brute_force(x, k, metric)
        out[f"{name}__index"] = idx
        out[f"{name}__dist_bits"] = dist.view(np.uint32)
        meta.append(dict(name=name, n=n, d=d, k=k, metric=metric, metric_id=METRICS[metric], seed=seed,
                         transform=transform, pairs=int(pairs)))
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(Path(__file__).with_name("golden.npz"), **out)
    print(f"wrote {len(CASES)} cases")


if __name__ == "__main__":
    main()
