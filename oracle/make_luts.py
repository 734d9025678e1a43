"""Generate the .splt approximation tables the path consumes as INPUT data.

The table build (optimize_knots per Lambda, lut.hpp:245-280) is out of scope
for the GPU path; the tables are produced here by the
reference's own deterministic ``build_lut(cubic_bspline(), {K, D}, N, {seed 0})``
through oracle/_ref and committed under data/luts/ (byte-deterministic given
the seed, lut_tests.cpp:216-226).  Run: ``python oracle/make_luts.py``.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "luts")

TABLES = [(4, 3, 1024), (4, 3, 16), (4, 3, 8), (3, 2, 64), (5, 4, 64), (2, 3, 64), (6, 6, 32),
          (7, 5, 32)] + [(K, D, 1024) for K in (1, 2, 3, 4) for D in (1, 2, 3)]


def main():
    os.makedirs(OUT, exist_ok=True)
    seen = set()
    for K, D, N in TABLES:
        if (K, D, N) in seen:
            continue
        seen.add((K, D, N))
        path = os.path.join(OUT, f"cubic_K{K}_D{D}_N{N}.splt")
        if os.path.exists(path):
            continue
        estar = ref.build_lut(K, D, N, path, seed=0, threads=0)
        print(f"K={K} D={D} N={N} E*={estar:.6e} -> {path}", flush=True)


if __name__ == "__main__":
    main()
