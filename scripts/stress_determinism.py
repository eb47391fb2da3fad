"""Re-solve golden cases repeatedly and compare histories bit for bit (the
iteration is deterministic by construction: fixed-order reductions), so any
difference between repeats exposes a race.  Usage on the GPU box:
    python scripts/stress_determinism.py [--reps 20] [--groups c5full,c2small]"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from golden_io import load_group  # noqa: E402
from test_gpu_parity import run_case  # noqa: E402


def sig(r):
    return [(h.sigma_star, h.residual) for h in r.history], r.iterations, r.status


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--groups", default="c5full,c2small,edge")
    ap.add_argument("--only", default="", help="comma list of case names")
    a = ap.parse_args()
    bad = 0
    total = 0
    for grp in a.groups.split(","):
        for name, g in load_group(grp).items():
            if a.only and name not in a.only.split(","):
                continue
            first = sig(run_case(g["case"]))
            for rep in range(a.reps):
                cur = sig(run_case(g["case"]))
                total += 1
                if cur != first:
                    bad += 1
                    h0, h1 = first[0], cur[0]
                    k = next((i for i in range(min(len(h0), len(h1))) if h0[i] != h1[i]), min(len(h0), len(h1)))
                    nd = sum(1 for i in range(min(len(h0), len(h1))) if h0[i] != h1[i])
                    nds = sum(1 for i in range(min(len(h0), len(h1))) if h0[i][0] != h1[i][0])
                    print(f"MISMATCH {grp}/{name} rep {rep}: iters {first[1]} vs {cur[1]}, first diff at record {k}: "
                          f"{h0[k] if k < len(h0) else None} vs {h1[k] if k < len(h1) else None}; "
                          f"{nd} records differ, {nds} in sigma*", flush=True)
    print(f"{bad} mismatching repeats of {total}")


if __name__ == "__main__":
    main()
