"""CPU tests of the drop-in boundary: libirgl_rt.so loads, exports every entry point that
include/irgl/rt.h declares, and its host-only planner (t_control) agrees with
a brute-force scan; without a GPU the runtime fails loudly (no CPU fallback)."""
import ctypes
import json
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "irgl", "rt.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)  # strip comments
    src = re.sub(r"//[^\n]*", "", src)
    return sorted(set(re.findall(r"\b(irgl_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_and_lib_exports_everything(irgl):
    syms = declared_symbols()
    assert len(syms) >= 20
    assert sorted(irgl.EXPORTS) == syms
    out = subprocess.check_output(["nm", "-D", "--defined-only", irgl.LIB_PATH]).decode()
    exported = set(re.findall(r" T (irgl_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing


def test_lib_is_sm100a_only(irgl):
    out = subprocess.run(["cuobjdump", "--list-elf", irgl.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_abi_version(irgl):
    assert irgl.load_library().irgl_abi_version() == 1


def brute_t_control(cs):
    dom = set(range(1, 1025))
    for kind, v in cs:
        if kind == 1:
            dom &= set(range(1, v + 1))
        elif kind == 2:
            dom &= {v}
    return max(dom) if dom else None


def test_t_control_golden_and_bruteforce(irgl):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))
    for cs, expect in gold["cases"]["t_control"]["cases"]:
        if expect is None:
            with pytest.raises(irgl.IrglError) as e:
                irgl.t_control([tuple(c) for c in cs])
            assert e.value.status == 6 and "outlining cannot be performed" in str(e.value)
        else:
            assert irgl.t_control([tuple(c) for c in cs]) == expect
    rng = np.random.default_rng(555)  # 1000 random constraint triples
    for _ in range(1000):
        cs = []
        for _ in range(3):
            k = int(rng.integers(0, 3))
            cs.append((k, int(rng.integers(1, 1025)) if k else 0))
        b = brute_t_control(cs)
        if b is None:
            with pytest.raises(irgl.IrglError):
                irgl.t_control(cs)
        else:
            assert irgl.t_control(cs) == b
            # permutation invariance; adding Elastic never changes the result
            assert irgl.t_control(cs[::-1]) == b
            assert irgl.t_control(cs + [(0, 0)]) == b


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly(irgl):
    with pytest.raises(irgl.IrglError) as e:
        irgl.Context()
    assert "no CUDA device" in str(e.value)


def test_invalid_arguments_are_values(irgl):
    L = irgl.load_library()
    assert L.irgl_ctx_create(None, -1, None, None) == 1  # IRGL_E_INVALID, no abort
    assert "E_INVALID" in L.irgl_last_error(None).decode()
    assert L.irgl_t_control(None, 0, None) == 1


def test_cpp_facade_compiles_and_links(irgl, tmp_path):
    """include/irgl/irgl.hpp (the C++ operator API over the C-ABI) builds against the .so."""
    src = os.path.join(ROOT, "examples", "bfs_listing2.cpp")
    exe = tmp_path / "bfs_listing2"
    subprocess.check_call(["/usr/bin/g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                           src, "-o", str(exe), "-L", os.path.dirname(irgl.LIB_PATH), "-lirgl_rt",
                           f"-Wl,-rpath,{os.path.dirname(irgl.LIB_PATH)}"])
    assert exe.exists()
