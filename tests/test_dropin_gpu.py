"""Drop-in by relinking: one host program written against the reference C ABI
(tests/dropin/dropin_demo.cpp: gt_greens_load, gt_field_load, gt_solve_steady with and
without the shift-variant term, gt_monte_carlo with a CSV) is compiled ONCE and linked
twice -- against the reference library built from its unchanged sources
(oracle/_ref/libgreentherm_ref.so) and against libgreentherm_b200.so -- and both binaries
run on the same files. Outputs agree to fp64 rounding."""
import csv
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _build(tmp_path, libdir, lib, name):
    exe = tmp_path / name
    obj = tmp_path / "dropin_demo.o"
    if not obj.exists():
        subprocess.run(["g++", "-std=c++17", "-O1", "-I", str(ROOT / "include"), "-c",
                        str(ROOT / "tests" / "dropin" / "dropin_demo.cpp"), "-o", str(obj)], check=True)
    subprocess.run(["g++", str(obj), "-L", str(libdir), f"-l:{lib}", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                   check=True)
    return exe


def _read_map(path):
    lines = path.read_text().split("\n")
    return np.array([[float(x) for x in l.split()] for l in lines[1:] if l.strip()])


def test_reference_program_relinks_unchanged(b200lib, oracle, greens64, tmp_path):
    import dataclasses
    from paper_2307_12119_b200 import inputs
    g = dataclasses.replace(greens64, rand_scale=2.0)
    oracle.save_greens_dir(g, tmp_path / "g")
    (tmp_path / "var.txt").write_text("beta 0.017\nseed 7\n")
    import ctypes as C
    f = C.c_void_p()
    assert b200lib.gt_field_create(64, g.pitch, b"watts", C.byref(f)) == 0
    np.ctypeslib.as_array(b200lib.gt_field_data(f), shape=(64, 64))[...] = \
        inputs.power_map(dataclasses.replace(inputs.CONFIGS["cfg0"], n=64), 5) * 0.3
    assert b200lib.gt_field_save(f, str(tmp_path / "p.map").encode()) == 0
    b200lib.gt_field_free(f)
    outs = {}
    for name, libdir, lib in (("ref", ROOT / "oracle" / "_ref", "libgreentherm_ref.so"),
                              ("b200", ROOT / "paper_2307_12119_b200", "libgreentherm_b200.so")):
        exe = _build(tmp_path, libdir, lib, f"demo_{name}")
        (tmp_path / name).mkdir()
        r = subprocess.run([str(exe), str(tmp_path / "g"), str(tmp_path / "var.txt"), str(tmp_path / "p.map"),
                            str(tmp_path / name) + "/"], capture_output=True, text=True, env={"GT_NO_BINARY_SIDECAR": "1"})
        assert r.returncode == 0, r.stderr
        outs[name] = r.stdout
        print(name, r.stdout)
    for m in ("steady.map", "steady_rand.map"):
        a, b = _read_map(tmp_path / "ref" / m), _read_map(tmp_path / "b200" / m)
        assert np.abs(a - b).max() <= 1e-8 * max(1.0, np.abs(a).max()), m
    ra = list(csv.DictReader(open(tmp_path / "ref" / "mc.csv")))
    rb = list(csv.DictReader(open(tmp_path / "b200" / "mc.csv")))
    assert [x["seed"] for x in ra] == [x["seed"] for x in rb]
    for x, y in zip(ra, rb):
        assert float(x["max_rise"]) == pytest.approx(float(y["max_rise"]), rel=1e-10)
        assert float(x["mean_rise"]) == pytest.approx(float(y["mean_rise"]), rel=1e-10)
