"""DMMA GEMM throughput on shapes the pipeline uses (tuning aid): TF/s and fraction of the
measured cuBLAS DGEMM (profiles/fp64_peaks_r01.json)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd  # noqa: E402

PEAK = 35.5
SHAPES = [  # (name, mode, M, N, K, batch)
    ("square4096_k512 (chol trailing)", 0, 4096, 4096, 512, 4),
    ("nt5800_k512 (chol trailing)", 2, 5184, 5184, 512, 8),
    ("nn5800_k64 (chol inner)", 2, 5184, 512, 64, 64),
    ("tn gram 400x400 k13800", 1, 400, 400, 13824, 64),
    ("nn S·Q 13800x386 k400", 0, 13824, 386, 400, 32),
    ("tn 300x300 k5184 (C2 gram)", 1, 300, 300, 5184, 256),
    ("tn 400x386 k13824 (C5 refine Sᵀ·Y)", 1, 400, 386, 13824, 64),
    ("nn 13824x213 k400 (C5 projection)", 0, 13824, 213, 400, 32),
    ("nn 1024^3", 0, 1024, 1024, 1024, 16),
    # the 80-wide CTA tile (mode + 10) on the m = 400 shapes
    ("tn gram 400x400 k13800, tile 80", 11, 400, 400, 13824, 64),
    ("nn S·Q 13800x386 k400, tile 80", 10, 13824, 386, 400, 32),
    ("tn 400x386 k13824, tile 80", 11, 400, 386, 13824, 64),
    ("nn 13824x213 k400, tile 80", 10, 13824, 213, 400, 32),
    ("nn S·Q 13800x386 k400, tile 64x80", 20, 13824, 386, 400, 32),
    ("nn 13824x213 k400, tile 64x80", 20, 13824, 213, 400, 32),
    ("nn 1280^3 tile 64x80", 20, 1280, 1280, 1280, 16),
    ("nn 1280^3 tile 64", 0, 1280, 1280, 1280, 16),
    ("nn 1280^3 tile 80", 10, 1280, 1280, 1280, 16),
    ("tn 1280^3 tile 64", 1, 1280, 1280, 1280, 16),
    ("tn 1280^3 tile 80", 11, 1280, 1280, 1280, 16),
]


def main():
    s = rdd.Solver(0)
    for name, mode, M, N, K, b in SHAPES:
        ms = s.bench_gemm(mode, M, N, K, b, reps=5)
        tf = 2.0 * M * N * K * b / (ms / 1e3) / 1e12
        print(json.dumps({"shape": name, "mode": mode, "M": M, "N": N, "K": K, "batch": b, "ms": ms,
                          "tflops": tf, "frac_of_cublas_dgemm": tf / PEAK}), flush=True)


if __name__ == "__main__":
    main()
