"""The reference's StitchEngine API (pipeline.hpp:341-721) on the drop-in:
tests/ref_unit/engine_bench.cpp compiled against the drop-in headers (whose
pipeline.hpp runs every frame on the device rig) and against the reference
headers (the CPU engine), on BASELINE configs 1 and 3. Composites must be
byte-identical between the builds and between Serial and Pipelined modes;
the frame rates are recorded next to the CPU engine's (gpurun_out/)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "ref_unit")


def _bin(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path) and os.path.isdir("/root/reference/proj/tests"):
        subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "tests", "ref_unit", "Makefile"), "all"],
                       check=True, cwd=ROOT)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    return path


def _run(name, *args):
    out = subprocess.run([_bin(name), *map(str, args)], capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def _record(tag, rows):
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"engine_dropin_{tag}.json"), "w") as f:
        json.dump(rows, f, indent=1)


def test_engine_bench_reference_cpu_runs():
    r = _run("engine_bench_ref", "cfg1", 2, "serial")
    assert r["frames"] == 2 and r["drops"] == 0


@pytest.mark.gpu
def test_stitch_engine_dropin_cfg1():
    ref = _run("engine_bench_ref", "cfg1", 20, "serial")
    ser = _run("engine_bench_b200", "cfg1", 300, "serial")
    pip = _run("engine_bench_b200", "cfg1", 300, "pipelined")
    short = _run("engine_bench_b200", "cfg1", 20, "serial")
    _record("cfg1", {"reference_cpu": ref, "b200_serial": ser, "b200_pipelined": pip})
    assert short["composite_fnv"] == ref["composite_fnv"] and short["composite_sum"] == ref["composite_sum"]
    assert short["first_fnv"] == ref["first_fnv"]
    assert ser["composite_fnv"] == pip["composite_fnv"]
    assert ser["estimations"] == pip["estimations"] == 300
    assert ser["drops"] == pip["drops"] == 0
    assert pip["frames_per_second"] >= 100 * ref["frames_per_second"], (pip, ref)


@pytest.mark.gpu
def test_stitch_engine_dropin_cfg3():
    ref = _run("engine_bench_ref", "cfg3", 1, "serial")
    ser = _run("engine_bench_b200", "cfg3", 40, "serial")
    pip = _run("engine_bench_b200", "cfg3", 40, "pipelined")
    _record("cfg3", {"reference_cpu": ref, "b200_serial": ser, "b200_pipelined": pip})
    assert ser["first_fnv"] == ref["first_fnv"] and ser["canvas"] == ref["canvas"]
    assert ser["composite_fnv"] == pip["composite_fnv"]
    assert ser["estimations"] == pip["estimations"] == 1
    assert pip["frames_per_second"] >= 100 * ref["frames_per_second"], (pip, ref)
