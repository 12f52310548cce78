"""CPU: the C-ABI library loads, exports every symbol include/heinfer_b200.h
declares, and its host-only entry points behave like the reference (no
device compute is called here)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2204_05496_b200 import ParamError, native, proposed_counts, baseline_counts, scale_value, RangeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "heinfer_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hei_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = native.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s
    assert set(native.EXPORTED) <= set(syms)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_closed_form_counts_through_abi():
    """test_matmul.cpp:293-324 through the C ABI."""
    assert proposed_counts(1, 1, 8, 8).as_tuple()[:3] == (2, 3, 4)
    c = proposed_counts(1, 11, 40960, 8192)
    assert (c.mul_plain_count, c.rotation_count, c.ciphertexts_in) == (66, 143, 5)
    c = proposed_counts(543, 11, 40960, 8192)
    assert c.mul_plain_count == 35838 and c.ciphertexts_out == 1
    assert baseline_counts(1, 11, 40960, 8192).mul_plain_count == 450560
    b1, b2, b3 = (baseline_counts(r, 11, 40960, 8192) for r in (1, 77, 8192))
    assert b1.mul_plain_count == b2.mul_plain_count == b3.mul_plain_count
    with pytest.raises(ParamError):
        proposed_counts(0, 1, 1, 8)
    with pytest.raises(ParamError):
        proposed_counts(1, 1, 1, 12)


def test_context_validation_before_any_device_work():
    """EncryptionParams::validate (params.cpp:27-66) errors surface as
    ParamError without touching a device."""
    from paper_2204_05496_b200 import GpuTwinServer

    q = [2147352577, 2147205121, 2147074049, 2146959361, 2146713601, 2146418689]
    with pytest.raises(ParamError):  # t1 = 114689 is not 1 mod 2n at n = 16384
        GpuTwinServer(16384, (1073872897, 114689), (6, 4), q + q[:4], [3], None)
    with pytest.raises(ParamError):  # not a power of two
        GpuTwinServer(12, (97, 17), (3, 3), q[:6], [3], None)
    with pytest.raises(ParamError):  # duplicate modulus
        GpuTwinServer(8192, (1073872897, 114689), (6, 4), q + [q[0], q[0], q[1], q[2]], [3], None)


def test_scale_value_matches_reference_rounding():
    """fixed_point.cpp:37-48 / test_fpcrt.cpp scale cases."""
    assert scale_value(1.5, 6) == 96
    assert scale_value(0.25, 14) == 4096
    assert scale_value(-0.5, 20) == -524288
    assert scale_value(0.0234375, 6) == 2
    assert scale_value(-0.0234375, 6) == -2
    # std::llround is half away from zero with no double rounding: the largest
    # double below 0.5 rounds to 0 (floor(|s| + 0.5) would give 1)
    assert scale_value(0.49999999999999994, 0) == 0
    assert scale_value(-0.49999999999999994, 0) == 0
    assert scale_value(2.5, 0) == 3
    assert scale_value(-2.5, 0) == -3
    assert scale_value(0.5, 0) == 1 and scale_value(-0.5, 0) == -1
    assert scale_value(1e13 + 0.5, 0) == 10000000000001 and scale_value(-(1e13 + 0.5), 0) == -10000000000001
    with pytest.raises(RangeError):
        scale_value(1e10, 20)
    with pytest.raises(RangeError):
        scale_value(float("nan"), 6)


def test_bench_q_chain_matches_reference_chain():
    import json

    import bench

    g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    assert bench.q_chain(8192, 1073872897) == g["chains"]["8192/1073872897/128"]
    assert bench.q_chain(8192, 114689) == g["chains"]["8192/114689/128"]
    assert bench.q_chain(16384, 163841) == g["chains"]["16384/163841/128"]


def test_device_prng_replays_reference_stream():
    """The product's util::Prng replay (host half) equals the reference stream."""
    from oracle.oracle import prng_stream
    from paper_2204_05496_b200 import Prng

    raw, _, _ = prng_stream(2, 1000)
    p = Prng(2)
    assert np.array_equal(p.draw(400), raw[:400])
    assert np.array_equal(p.draw(600), raw[400:])


def test_null_context_is_a_param_error_not_a_crash():
    """Every C entry point validates its context before any device work."""
    import ctypes as C

    lib = native.lib()
    out = np.zeros(4, np.uint64)
    assert lib.hei_gpu_matmul(None, None, None, 1, C.c_uint64(1), None, None, None) == native.HEI_PARAM_ERROR
    assert lib.hei_gpu_upload_public_key(None, C.c_uint32(0), native.u64p(out)) in (native.HEI_PARAM_ERROR,)
    assert b"null context" in lib.hei_gpu_last_error()
