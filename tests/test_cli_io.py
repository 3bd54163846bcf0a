"""ArrayFile I/O, strict JSON config and the CLI (CPU: no device needed for
I/O and config; the recon command itself is covered in test_gpu_solver.py).

Fixtures tests/golden/arrayio_*.hicu were written by the reference's
`arrayio.write_array` (tests/golden/make_arrayio.py)."""

import json
import os

import numpy as np
import pytest

import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import cli
from paper_2004_08962_b200.errors import ArrayFormatError, ConfigError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("key", ["c16", "f8", "u1"])
def test_reads_reference_files_and_writes_identical_bytes(tmp_path, key):
    ref = np.load(os.path.join(GOLD, "arrayio_ref.npz"))[key]
    path = os.path.join(GOLD, f"arrayio_{key}.hicu")
    got = H.read_array(path)
    assert got.dtype == ref.dtype and got.shape == ref.shape
    assert np.array_equal(got, ref)
    out = tmp_path / "x.hicu"
    H.write_array(out, ref)
    assert out.read_bytes() == open(path, "rb").read()


def test_round_trip_bit_exact_and_dtype_mapping(tmp_path):
    rng = np.random.default_rng(0)
    p = tmp_path / "a.hicu"
    c64 = (rng.standard_normal((4, 3)) + 1j * rng.standard_normal((4, 3))).astype(np.complex64)
    H.write_array(p, c64)
    back = H.read_array(p)
    assert back.dtype == np.complex128 and np.array_equal(back, c64.astype(np.complex128))
    H.write_array(p, np.array([[True, False]]))
    assert H.read_array(p).dtype == np.uint8
    H.write_array(p, np.arange(3, dtype=np.float32))
    assert H.read_array(p).dtype == np.float64


def test_format_errors(tmp_path):
    p = tmp_path / "bad.hicu"
    with pytest.raises(ArrayFormatError):
        H.write_array(p, np.array([0, 2], np.uint8))  # mask must be {0,1}
    with pytest.raises(ArrayFormatError):
        H.write_array(p, np.array(["a"]))
    good = open(os.path.join(GOLD, "arrayio_f8.hicu"), "rb").read()
    for blob in (good[:5], b"XXXX" + good[4:], good[:4] + bytes([2]) + good[5:],
                 good[:5] + bytes([9]) + good[6:], good[:6] + bytes([0]) + good[7:], good[:12], good + b"\x00"):
        p.write_bytes(blob)
        with pytest.raises(ArrayFormatError):
            H.read_array(p)


def _doc():
    return {"seed": 3, "kernel": {"extents": [5, 5, 4]},
            "schedule": {"rank": 20, "stages": [{"region": [0.5, 0.5, "full"], "p": 4, "gradient_steps": 2,
                                                 "iterations": 3},
                                                {"region": "full", "p": 4, "gradient_steps": 2, "iterations": 2}],
                         "dc_mode": "soft", "dc_lambda": 0.3, "seed": 9},
            "metrics": {"ssim": False},
            "paths": {"kspace": "k.hicu", "mask": "m.hicu"},
            "phantom": {"nx": 32, "ny": 32, "ncoils": 4, "ellipses": [
                {"center": [0, 0], "axes": [0.3, 0.2], "intensity": 1.0}]},
            "mask": {"pattern": "vd_1d", "r": 3}}


def test_config_parses_reference_schema():
    cfg = H.parse_config(_doc())
    assert cfg.seed == 3 and cfg.kernel.n == 100
    sc = cfg.schedule
    assert sc.rank == 20 and sc.dc_mode == "soft" and sc.dc_lambda == 0.3 and sc.seed == 9
    assert sc.stages[0].region == [0.5, 0.5, "full"] and sc.stages[1].region == "full"
    assert cfg.metrics == {"ssim": False, "hfen": True, "ssos": False}
    ell = H.parse_config({"kernel": {"extents": [5, 5, 4], "shape": "ellipsoid"}}).kernel
    assert ell.n < 100


@pytest.mark.parametrize("mutate", [
    lambda d: d.update(bogus=1),
    lambda d: d["schedule"].update(typo=1),
    lambda d: d["schedule"]["stages"][0].pop("p"),
    lambda d: d["schedule"]["stages"][0].update(region=[True, 0.5, "full"]),
    lambda d: d["schedule"]["stages"][1].update(region="half"),
    lambda d: d["kernel"].update(shape="star"),
    lambda d: d["paths"].update(output="x"),
    lambda d: d["phantom"]["ellipses"][0].update(color="red"),
    lambda d: d["mask"].pop("r"),
    lambda d: d["metrics"].update(psnr=True),
])
def test_config_rejects_unknown_and_missing(mutate):
    d = _doc()
    mutate(d)
    with pytest.raises(ConfigError):
        H.parse_config(d)


def test_load_config_errors(tmp_path):
    p = tmp_path / "c.json"
    p.write_text("{not json")
    with pytest.raises(ConfigError):
        H.load_config(p)
    p.write_text("[1, 2]")
    with pytest.raises(ConfigError):
        H.load_config(p)


def test_cli_errors_and_metrics(tmp_path, capsys):
    cfgp = tmp_path / "c.json"
    cfgp.write_text(json.dumps(_doc()))
    assert cli.main(["recon"]) == 2                                   # recon requires --config
    assert cli.main(["phantom", "--config", str(cfgp)]) == 2          # simulator not in the B200 build
    assert cli.main(["recon", "--config", str(cfgp), "--out", str(tmp_path)]) == 2  # inputs missing
    assert "input file does not exist" in capsys.readouterr().err
    rng = np.random.default_rng(1)
    ref = rng.standard_normal((8, 8, 2)) + 1j * rng.standard_normal((8, 8, 2))
    H.write_array(tmp_path / "r.hicu", ref)
    H.write_array(tmp_path / "e.hicu", ref * 1.01)
    assert cli.main(["metrics", str(tmp_path / "r.hicu"), str(tmp_path / "e.hicu"), "--ssos"]) == 0
    out = capsys.readouterr().out
    assert "SER: 40.00 dB" in out and "SSoS SER: 40.00 dB" in out
    H.write_array(tmp_path / "e2.hicu", ref[:4])
    assert cli.main(["metrics", str(tmp_path / "r.hicu"), str(tmp_path / "e2.hicu")]) == 2
