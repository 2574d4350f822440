"""CPU-side checks of the native product (no GPU needed):

* the C-ABI libraries load and export every symbol the headers declare;
* the host C++ API (scheduler, cost model, simulator, profile/schedule I/O)
  is byte-identical to the REAL reference — fixtures and fuzzed instances —
  through the same parity_tool source compiled against both libraries;
* the reference's own acceptance binary, compiled against this library,
  passes its host-only criteria;
* the device path fails loudly (no silent CPU fallback) without a GPU.
"""
import os
import re
import subprocess

import pytest

from tests import golden_io as G

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(REPO, "build", "parity_tool")
REF_TOOL = os.path.join(REPO, "oracle", "_ref", "parity_tool_ref")
ACCEPT = os.path.join(REPO, "build", "acceptance")


def _declared(header, prefix):
    text = open(os.path.join(REPO, "include", header)).read()
    return sorted(set(re.findall(r"\b(" + prefix + r"_\w+)\s*\(", text)))


def _exports(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if ln.strip()}


@pytest.mark.parametrize("header", ["dsx.h", "dsx_nn.h"])
def test_dsx_exports_every_declared_symbol(header):
    from paper_2502_11058_b200 import native
    declared = _declared(header, "dsx")
    assert declared == native.exported_symbols(header)
    exported = _exports(native.DSX_PATH)
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    native.load_dsx()  # resolves every signature


def test_dense_gemm_uses_tcgen05_and_tma():
    """The NN layer GEMMs are tcgen05 (UTCHMMA, TMEM loads) fed by TMA
    (UTMALDG) — checked in the SASS of the shipped library."""
    from paper_2502_11058_b200 import native
    out = subprocess.run(["cuobjdump", "-sass", native.DSX_PATH], capture_output=True, text=True).stdout
    for op in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert op in out, op


def test_dreamsched_c_exports():
    from paper_2502_11058_b200 import native
    declared = _declared("dreamsched_c.h", "dsc")
    exported = _exports(native.DREAMSCHED_PATH)
    assert declared and all(s in exported for s in declared)


def test_kernels_target_sm100a():
    from paper_2502_11058_b200 import native
    out = subprocess.run(["cuobjdump", "--list-elf", native.DSX_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def run_tool(*args):
    return subprocess.run([TOOL] + list(args), check=True, capture_output=True, text=True).stdout


def test_sched_fuzz_golden_byte_identical():
    assert run_tool("sched-fuzz", "2026", "150", "40") == G.read("sched_fuzz_2026.txt")


@pytest.mark.parametrize("name,h", [("resnet18_like", 5), ("three_layer", 2),
                                    ("three_layer_light", 2), ("totals_123", 1),
                                    ("mlp8_w1024", 4)])
def test_profile_fixture_schedules_byte_identical(name, h):
    out = run_tool("profile", os.path.join(G.DATA, name + ".profile"), str(h))
    assert out.replace(G.DATA + "/", "") == G.read("profile_%s_h%d.txt" % (name, h))


def test_trace_json_byte_identical():
    out = run_tool("trace", os.path.join(G.DATA, "three_layer.profile"), "plsgd", "2", "2")
    assert out == G.read("trace_three_layer_plsgd.txt")


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="reference build absent")
@pytest.mark.parametrize("L,seed", [(12, 1), (24, 7), (36, 3), (48, 11)])
def test_synth_profile_sweep_inputs_match_reference(L, seed):
    """synth_profile (the schedule sweep's generator) and its DFS + fill
    schedules, byte-identical to the reference for every regime."""
    ref = subprocess.run([REF_TOOL, "synth", str(L), str(seed)], check=True, capture_output=True,
                         text=True).stdout
    assert run_tool("synth", str(L), str(seed)) == ref


def test_c_abi_synth_profile(tmp_path):
    import ctypes as C

    from paper_2502_11058_b200 import native
    from paper_2502_11058_b200.lab import _dsc
    native.load_dsx()
    path = str(tmp_path / "s.profile")
    assert _dsc().dsc_synth_profile(path.encode(), C.c_int(12), C.c_uint64(1), b"balanced") == 0
    assert open(path).read() == run_tool("synth", "12", "1").split("dreamsched-schedule")[0]
    assert _dsc().dsc_synth_profile(path.encode(), C.c_int(12), C.c_uint64(1), b"bogus") == 1


def test_c_abi_simulator_matches_trace_fixture():
    """dsc_simulate_trace + dsc_compare_modes (the C-ABI the four-mode GPU
    runner uses) reproduce the reference's trace + mode report byte for byte."""
    from paper_2502_11058_b200 import modes
    prof = os.path.join(G.DATA, "three_layer.profile")
    makespan, trace = modes.simulate(prof, "plsgd", 2, 2)
    assert trace + modes.compare(prof, 2, 2) == G.read("trace_three_layer_plsgd.txt")
    assert makespan == 9.0


def test_measured_trace_schema_matches_simulator():
    """The measured-timeline export uses the simulator's trace schema."""
    import json

    import numpy as np

    from paper_2502_11058_b200 import modes
    # one step, 2 layers: BP L2 [0,1] ms, BP L1 [1,2] ms, COMM L1 [2,4] ms
    bp = np.array([1.0, 2.0, 0.0, 1.0], dtype=np.float32)
    comm = np.array([2.0, 4.0, -1.0, -1.0], dtype=np.float32)
    got = json.loads(modes.trace_json("plsgd", [(bp, comm)]))
    sim = json.loads(modes.simulate(os.path.join(G.DATA, "three_layer.profile"), "plsgd", 2, 2)[1])
    assert {tuple(sorted(e)) for e in got} == {tuple(sorted(e)) for e in sim if "layer" in e["args"]}
    assert [(e["name"], e["ts"], e["dur"], e["tid"]) for e in got] == [
        ("BP L2", 0, 1000, "compute"), ("BP L1", 1000, 1000, "compute"), ("COMM L1", 2000, 2000, "link")]


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="reference build absent")
@pytest.mark.parametrize("seed,count,maxl", [(11, 600, 24), (12, 300, 61)])
def test_sched_fuzz_live_against_reference(seed, count, maxl):
    args = ["sched-fuzz", str(seed), str(count), str(maxl)]
    ref = subprocess.run([REF_TOOL] + args, check=True, capture_output=True, text=True).stdout
    assert run_tool(*args) == ref


@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 5, 10])
def test_reference_acceptance_host_criteria(criterion):
    if not os.path.exists(ACCEPT):
        pytest.skip("acceptance binary is built only where /root/reference exists")
    out = subprocess.run([ACCEPT, "--only", str(criterion)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "[PASS]" in out.stdout


def test_device_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2502_11058_b200 import DsxError, Lab, LabDesc
    with pytest.raises(DsxError):
        Lab(LabDesc(dim=16, block_sizes=[8, 8], workers_total=2))
    out = subprocess.run([TOOL, "steps", "12", "3", "4", "3", "0.5", "7", "1", "partial", "enp"],
                         capture_output=True, text=True)
    assert out.returncode != 0 and "dsx_lab_create" in out.stderr


@pytest.mark.parametrize("jump", [1, 311, 312, 19936, 19937, 100003, 2000000])
def test_mt_jump_ahead_matches_recurrence(jump):
    """The GF(2) characteristic-polynomial jump used by the parallel noise
    engine equals running std::mt19937_64's recurrence (host-only)."""
    import ctypes as C
    from paper_2502_11058_b200 import native
    ok = C.c_int(0)
    native.call("dsx_mt_jump_selftest", jump, C.byref(ok))
    assert ok.value == 1


def test_sweep_layer_sizes_follow_synth_profile():
    """tools/sweep.py scales synth_profile's layer bytes to the requested
    per-worker dimension (even sizes, every layer >= 2 coordinates)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("sweep", os.path.join(REPO, "tools", "sweep.py"))
    sweep = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sweep)
    from paper_2502_11058_b200.lab import profile_layers
    sizes = sweep.synth_sizes(24, 1, "balanced", 1_000_000, 0)
    assert len(sizes) == 24 and all(s >= 2 and s % 2 == 0 for s in sizes)
    assert abs(sum(sizes) - 1_000_000) <= 2 * 24
    # proportional to the profile's bytes
    import subprocess as sp
    text = sp.run([TOOL, "synth", "24", "1"], check=True, capture_output=True, text=True).stdout
    pb = [int(ln.split("\t")[2]) for ln in text.split("dreamsched-schedule")[0].splitlines()[1:25]]
    big = max(range(24), key=lambda i: pb[i])
    assert sizes[big] == max(sizes)
    del profile_layers
