"""CPU: config parsing / validation of the GPU-backend CLI (mirrors the
reference cli.py:92-262 schema checks and exit codes), the phase-map files
(P-PHASE raster, geometry.py:126-189; bit-packed binary), and the byte
format of the artifact writers.  No device work."""

from __future__ import annotations

import textwrap

import numpy as np
import pytest

import paper_2001_08289_b200 as fb
from paper_2001_08289_b200 import cli


def _cfg(tmp_path, text, name="run.cfg"):
    p = tmp_path / name
    p.write_text(textwrap.dedent(text))
    return p


BASE = """
[geometry]
kind = square
n = 16
side_fraction = 0.5

[physics]
sigma1_re = 2.0

[scheme]
name = em_sub
alpha = 0.25
beta = 4.0
tol = 1e-10
"""


def test_parse_and_echo(tmp_path):
    cfg = cli.parse_config(_cfg(tmp_path, BASE))
    assert cfg.geometry == {"kind": "square", "n": 16, "side_fraction": 0.5}
    assert cfg.physics == {"sigma1_re": 2.0, "sigma1_im": 0.0}
    assert cfg.scheme == {"name": "em_sub", "alpha": 0.25, "beta": 4.0, "tol": 1e-10, "max_iters": 1000}
    sc = cli._solver_config(cfg, "em_sub", 2)
    assert sc.sigma1 == 2.0 and sc.e0 == (1.0, 0.0) and sc.interval.beta == 4.0


def test_overrides_and_extended_keys(tmp_path):
    cfg = cli.parse_config(_cfg(tmp_path, BASE), ["geometry.dim=3", "physics.e0=1, 1j, 0.5", "scheme.max_iters=7"])
    assert cfg.geometry["dim"] == 3 and cfg.scheme["max_iters"] == 7
    assert cfg.physics["e0"] == [[1.0, 0.0], [0.0, 1.0], [0.5, 0.0]]
    sc = cli._solver_config(cfg, "em_sub", 3)
    assert sc.e0 == (1.0, 1j, 0.5)
    pm = cli.build_phase_map(cfg)
    assert pm.grid == (16, 16, 16) and int(pm.chi.sum()) == 8 ** 3
    with pytest.raises(fb.ConfigError):
        cli._solver_config(cfg, "em_sub", 2)  # 3 components on a 2-D cell


@pytest.mark.parametrize("patch, msg", [
    (["bogus.key=1"], "unknown section"),
    (["geometry.colour=red"], "unknown key"),
    (["geometry.kind=hexagon"], "kind must be"),
    (["scheme.names=basic,em"], "either name or names"),
    (["scheme.tol=-1"], "tol must be positive"),
    (["scheme.max_iters=0"], "max_iters"),
    (["scheme.alpha=5.0"], "bad interval"),
    (["physics.e0=1,2,3,4"], "2 or 3 components"),
    (["physics.e0=0,0"], "nonzero"),
    (["physics.e0=a,b"], "complex"),
    (["geometry.kind=cube"], "cube needs side"),
    (["geometry.kind=random"], "random needs"),
    (["geometry.dim=4"], "dim must be"),
    (["noequals"], "override must look like"),
])
def test_config_errors(tmp_path, patch, msg):
    path = _cfg(tmp_path, BASE)
    if patch == ["geometry.kind=cube"] or patch == ["geometry.kind=random"]:
        text = BASE.replace("side_fraction = 0.5\n", "")
        path = _cfg(tmp_path, text, "b.cfg")
    with pytest.raises(fb.ConfigError, match=msg):
        cli.parse_config(path, patch)


def test_main_exit_code_2_on_config_error(tmp_path, capsys):
    rc = cli.main(["solve", str(_cfg(tmp_path, BASE)), "--override", "scheme.name=nope"])
    assert rc == 2
    assert "unknown scheme" in capsys.readouterr().err


def test_geometry_kinds(tmp_path):
    cube = cli.parse_config(_cfg(tmp_path, BASE), ["geometry.kind=cube", "geometry.side=6"])
    assert cli.build_phase_map(cube).grid == (16, 16, 16)
    rnd = cli.parse_config(_cfg(tmp_path, BASE), ["geometry.kind=random", "geometry.dim=3", "geometry.seed=3",
                                                   "geometry.smoothing=1.5", "geometry.fraction=0.3"])
    pm = cli.build_phase_map(rnd)
    assert pm.grid == (16, 16, 16) and abs(float(pm.volume_fraction) - 0.3) < 0.01
    fb.save_chi_bits(pm, tmp_path / "m.chi")
    bits = cli.parse_config(_cfg(tmp_path, BASE), ["geometry.kind=bits", "geometry.path=m.chi"])
    assert cli.build_phase_map(bits) == pm
    (tmp_path / "r.txt").write_text(fb.save_raster(fb.build_disk_array(8, 0.3)))
    ras = cli.parse_config(_cfg(tmp_path, BASE), ["geometry.kind=raster", "geometry.path=r.txt"])
    assert cli.build_phase_map(ras) == fb.build_disk_array(8, 0.3)
    bad = cli.parse_config(_cfg(tmp_path, BASE), ["geometry.side_fraction=0.3"])
    with pytest.raises(fb.ConfigError, match="geometry"):
        cli.build_phase_map(bad)


def test_raster_round_trip_and_errors():
    pm = fb.build_square_array(8, 0.5)
    text = fb.save_raster(pm)
    assert text.splitlines()[0] == "P-PHASE 8 8"
    assert fb.load_raster(text) == pm
    with pytest.raises(fb.RasterParseError) as e:
        fb.load_raster("P-PHASE 4 2\n0 1 0 1\n0 2 0 1\n")
    assert e.value.line == 3 and e.value.column == 2
    with pytest.raises(fb.RasterParseError):
        fb.load_raster("P-PHASE 3 2\n")
    with pytest.raises(fb.RasterParseError) as e:
        fb.load_raster("P-PHASE 2 2\n0 1\n1 0\nextra\n")
    assert e.value.line == 4


@pytest.mark.parametrize("shape", [(6, 10), (4, 6, 10), (2, 2)])
def test_chi_bits_round_trip(tmp_path, shape):
    rng = np.random.default_rng(1)
    pm = fb.PhaseMap(rng.random(shape) < 0.5)
    fb.save_chi_bits(pm, tmp_path / "a.chi")
    raw = (tmp_path / "a.chi").read_bytes()
    assert raw[:8] == b"FFTCHI01" and len(raw) == 40 + (int(np.prod(shape)) + 7) // 8
    assert fb.load_chi_bits(tmp_path / "a.chi") == pm
    (tmp_path / "b.chi").write_bytes(b"NOTACHI0" + raw[8:])
    with pytest.raises(fb.RasterParseError):
        fb.load_chi_bits(tmp_path / "b.chi")
    (tmp_path / "c.chi").write_bytes(raw[:-1])
    with pytest.raises(fb.RasterParseError):
        fb.load_chi_bits(tmp_path / "c.chi")


def test_history_csv_bytes(tmp_path):
    h = fb.ConvergenceHistory()
    h.append(1, 1.8035714285714286 + 0j, 0.5)
    h.append(2, 1.25 - 1e-20j, 1e-11)
    res = fb.SolveResult(sigma_star=h.records[-1].sigma_star, E_field=None, J_field=None, history=h,
                         status=fb.TerminationStatus.CONVERGED, degenerate_flux=False, mean_E=None, mean_J=None,
                         device_ms=0.0)
    cli._write_history_csv(tmp_path / "h.csv", res)
    assert (tmp_path / "h.csv").read_bytes() == (
        b"iter,sigma_star_re,sigma_star_im,residual\n"
        b"1,1.8035714285714286,0,0.5\n"
        b"2,1.25,-9.9999999999999995e-21,9.9999999999999994e-12\n")


def test_obnosov_and_predicted_rate(tmp_path):
    assert cli.obnosov(1.0) == 1.0
    assert abs(cli.obnosov(0.0) - 1 / 3 ** 0.5) < 1e-15
    cfg = cli.parse_config(_cfg(tmp_path, BASE))
    z = fb.map_z(fb.SchemeKind.EYRE_MILTON_SUB, 2.0, fb.SpectralInterval(0.25, 4.0))
    assert cli._predicted_rate_or_none(cfg, "em_sub") == abs(z)
    assert cli._exact_reference(cfg) == cli.obnosov(2.0)
