"""Golden CLI artifacts from the LIVE reference CLI (TEST INFRASTRUCTURE;
dev container only).  Runs ``fftcond.cli.main`` (reference cli.py:448-478)
on a few configurations and freezes the artifacts it writes (history CSVs,
result JSON, compare summary CSV) plus its exit code and stdout under
tests/golden/cli/<case>/.  The config texts are written here (values of the
reference's shipped benchmark/compare configs and variations).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_cli.py
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import shutil
import sys

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from fftcond import cli as RCLI  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "cli")

CASES = {
    # insulating square array, em_sub against the exact value 1/sqrt(3)
    "benchmark": ("solve", """[geometry]
kind = square
n = 128
side_fraction = 0.5

[physics]
sigma1_re = 0.0

[scheme]
name = em_sub
alpha = 0.25
beta = 4.0
tol = 2e-3
max_iters = 200

[output]
history_csv = history.csv
result_json = result.json
"""),
    # all four schemes, exact reference applied automatically
    "compare": ("compare", """[geometry]
kind = square
n = 128
side_fraction = 0.5

[physics]
sigma1_re = 2.0

[scheme]
names = basic, em, basic_sub, em_sub
alpha = 0.25
beta = 4.0
tol = 1e-10
max_iters = 1000

[output]
history_csv = history.csv
summary_csv = summary.csv
"""),
    # complex sigma1, sigma0 override, disk geometry, MaxIters exit
    "disk_complex": ("solve", """[geometry]
kind = disk
n = 64
radius = 0.3

[physics]
sigma1_re = 5.0
sigma1_im = 2.0

[scheme]
name = em
tol = 1e-12
max_iters = 40
sigma0_re = 2.5
sigma0_im = 0.5

[output]
history_csv = history.csv
result_json = result.json
"""),
    # grids outside the fused power-of-two lengths (the general cuFFT path)
    "compare_n96": ("compare", """[geometry]
kind = square
n = 96
side_fraction = 0.5

[physics]
sigma1_re = 2.0

[scheme]
names = basic, em, basic_sub, em_sub
alpha = 0.25
beta = 4.0
tol = 1e-10
max_iters = 1000

[output]
history_csv = history.csv
summary_csv = summary.csv
"""),
    "disk_n100": ("solve", """[geometry]
kind = disk
n = 100
radius = 0.3

[physics]
sigma1_re = 5.0
sigma1_im = 2.0

[scheme]
name = em_sub
alpha = 0.25
beta = 4.0
tol = 1e-10
max_iters = 1000

[output]
history_csv = history.csv
result_json = result.json
"""),
    # a scheme that errors (branch cut) inside compare
    "compare_branch_cut": ("compare", """[geometry]
kind = square
n = 32
side_fraction = 0.5

[physics]
sigma1_re = -2.0

[scheme]
names = basic, em
tol = 1e-8
max_iters = 50

[output]
summary_csv = summary.csv
"""),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    only = set(sys.argv[1:])
    for name, (cmd, text) in CASES.items():
        if only and name not in only:
            continue
        d = os.path.join(OUT, name)
        shutil.rmtree(d, ignore_errors=True)
        os.makedirs(d)
        with open(os.path.join(d, "run.cfg"), "w") as fh:
            fh.write(text)
        out, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            rc = RCLI.main([cmd, os.path.join(d, "run.cfg")])
        with open(os.path.join(d, "meta.json"), "w") as fh:
            json.dump({"command": cmd, "exit_code": rc, "stdout": out.getvalue(), "stderr": err.getvalue()}, fh,
                      indent=1)
        print(name, rc, sorted(os.listdir(d)))


if __name__ == "__main__":
    main()
