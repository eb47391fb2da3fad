"""GPU: the CLI on the B200 backend against artifacts of the live reference
CLI (tests/golden/cli, oracle/gen_golden_cli.py): exit codes, per-scheme
status and iteration counts identical; sigma* histories within 1e-10
relative and residuals within 1e-4 (SURVEY 8(c) parity protocol); config
echo and predicted rates identical; artifacts byte-deterministic run to
run.  Plus the 3-D / e0 / bit-packed-chi extensions against the oracle."""

from __future__ import annotations

import contextlib
import io
import json
import os
import shutil

import numpy as np
import pytest

from golden_io import GOLDEN

pytestmark = pytest.mark.gpu

CLI_GOLD = os.path.join(GOLDEN, "cli")
CASES = sorted(os.listdir(CLI_GOLD)) if os.path.isdir(CLI_GOLD) else []


def _run(args):
    from paper_2001_08289_b200 import cli

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(args)
    return rc, out.getvalue(), err.getvalue()


def _hist(path):
    rows = open(path).read().splitlines()
    assert rows[0] == "iter,sigma_star_re,sigma_star_im,residual"
    return np.array([[float(x) for x in r.split(",")] for r in rows[1:]]).reshape(-1, 4)


def _check_hist(got, want):
    assert got.shape == want.shape
    assert np.array_equal(got[:, 0], want[:, 0])
    gs, ws = got[:, 1] + 1j * got[:, 2], want[:, 1] + 1j * want[:, 2]
    assert np.all(np.abs(gs - ws) <= 1e-10 * np.abs(ws))
    assert np.all(np.abs(got[:, 3] - want[:, 3]) <= 1e-4 * np.abs(want[:, 3]) + 1e-16)


def _parse_lines(text):
    out = {}
    for line in text.splitlines():
        name, rest = line.split(": ", 1)
        if rest.startswith("error"):
            out[name] = ("error", None, None)
            continue
        status, rest = rest.split(" after ")
        iters = int(rest.split(" ")[0])
        sigma = complex(rest.split("sigma_star = ")[1])
        out[name] = (status, iters, sigma)
    return out


@pytest.mark.parametrize("case", CASES)
def test_cli_matches_reference_cli(case, tmp_path):
    src = os.path.join(CLI_GOLD, case)
    meta = json.load(open(os.path.join(src, "meta.json")))
    work = tmp_path / case
    work.mkdir()
    shutil.copy(os.path.join(src, "run.cfg"), work / "run.cfg")
    rc, out, _ = _run([meta["command"], str(work / "run.cfg")])
    assert rc == meta["exit_code"]
    got, want = _parse_lines(out), _parse_lines(meta["stdout"])
    assert got.keys() == want.keys()
    for k in want:
        assert got[k][:2] == want[k][:2], k
        if want[k][2] is not None:
            assert abs(got[k][2] - want[k][2]) <= 1e-9 * abs(want[k][2]), k
    for fn in sorted(os.listdir(src)):
        if fn.startswith("history"):
            _check_hist(_hist(work / fn), _hist(os.path.join(src, fn)))
    if os.path.exists(os.path.join(src, "result.json")):
        g, w = json.load(open(work / "result.json")), json.load(open(os.path.join(src, "result.json")))
        assert (g["status"], g["iterations"], g["config"], g["predicted_rate"]) == \
               (w["status"], w["iterations"], w["config"], w["predicted_rate"])
        gs, ws = complex(g["sigma_star"]["re"], g["sigma_star"]["im"]), complex(w["sigma_star"]["re"], w["sigma_star"]["im"])
        assert abs(gs - ws) <= 1e-10 * abs(ws)
        if w["estimated_rate"] is None:
            assert g["estimated_rate"] is None
        else:
            assert abs(g["estimated_rate"] - w["estimated_rate"]) <= 1e-4 * w["estimated_rate"]
    if os.path.exists(os.path.join(src, "summary.csv")):
        grows = [r.split(",") for r in open(work / "summary.csv").read().splitlines()]
        wrows = [r.split(",") for r in open(os.path.join(src, "summary.csv")).read().splitlines()]
        assert grows[0] == wrows[0] and len(grows) == len(wrows)
        for g, w in zip(grows[1:], wrows[1:]):
            assert g[:3] == w[:3] and g[5] == w[5]
            if w[3]:
                assert abs(float(g[3]) - float(w[3])) <= max(1e-9, 1e-10 * abs(float(w[3])))
            if w[4]:
                assert abs(float(g[4]) - float(w[4])) <= 1e-4 * float(w[4])
    # byte determinism: a second run writes identical artifacts
    first = {fn: (work / fn).read_bytes() for fn in os.listdir(work) if fn != "run.cfg"}
    rc2, out2, _ = _run([meta["command"], str(work / "run.cfg")])
    assert (rc2, out2) == (rc, out)
    assert {fn: (work / fn).read_bytes() for fn in first} == first


def test_cli_3d_cube_e0_and_bits(tmp_path):
    import paper_2001_08289_b200 as fb
    from oracle import fftcond_oracle as O

    pm = fb.build_random_medium(16, 3, seed=5, smoothing=1.5, fraction=0.3)
    fb.save_chi_bits(pm, tmp_path / "medium.chi")
    (tmp_path / "r.cfg").write_text(
        "[geometry]\nkind = bits\npath = medium.chi\n\n[physics]\nsigma1_re = 50.0\ne0 = 0.5773502691896258, "
        "0.5773502691896258, 0.5773502691896258\n\n[scheme]\nname = em_sub\nalpha = 0.25\nbeta = 4.0\n"
        "tol = 1e-8\n\n[output]\nhistory_csv = h.csv\nresult_json = r.json\nfields_npz = f.npz\n")
    rc, out, err = _run(["solve", str(tmp_path / "r.cfg")])
    assert rc == 0, err
    e0 = (0.5773502691896258,) * 3
    ref = O.solve(pm.chi, "em_sub", 50.0, e0=e0, tol=1e-8, alpha=0.25, beta=4.0)
    h = _hist(tmp_path / "h.csv")
    assert len(h) == len(ref.history)
    assert abs(complex(h[-1, 1], h[-1, 2]) - ref.sigma_star) <= 1e-10 * abs(ref.sigma_star)
    z = np.load(tmp_path / "f.npz")
    assert z["E"].shape == (3, 16, 16, 16) and np.array_equal(z["chi"], pm.chi)
    cube = tmp_path / "c.cfg"
    cube.write_text("[geometry]\nkind = cube\nn = 16\nside = 8\n\n[physics]\nsigma1_re = 10.0\ne0 = 0, 0, 1\n\n"
                    "[scheme]\nname = basic\ntol = 1e-8\n\n[output]\nresult_json = c.json\n")
    rc, out, err = _run(["solve", str(cube)])
    assert rc == 0, err
    ref = O.solve(fb.build_cube_array(16, 8).chi, "basic", 10.0, e0=(0, 0, 1), tol=1e-8)
    r = json.load(open(tmp_path / "c.json"))
    assert r["iterations"] == len(ref.history)
    assert abs(complex(r["sigma_star"]["re"], r["sigma_star"]["im"]) - ref.sigma_star) <= 1e-10 * abs(ref.sigma_star)


def test_cli_selftest_command():
    from paper_2001_08289_b200 import selftest
    from paper_2001_08289_b200.exceptions import BackendError

    try:
        selftest.reference_module()
    except BackendError:
        pytest.skip("reference package not installed (baseline/_ref)")
    rc, out, _ = _run(["selftest"])
    assert rc == 0 and out.endswith("13/13 checks passed\n")
