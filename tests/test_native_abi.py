"""CPU checks of the C ABI boundary and of the device curve math compiled for the host."""

import ctypes
import os
import re
import subprocess
import shutil

import numpy as np
import pytest

import golden_io as gio
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tokencarve_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|int)\s+(tcb_\w+)\s*\(", text, re.M)))


def test_library_builds_and_exports_every_header_symbol():
    from paper_2505_16864_b200 import _build, _native

    lib_path = _build.build()
    lib = ctypes.CDLL(lib_path)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.SIGNATURES), "ctypes table must mirror the header"
    assert _native.load().tcb_abi_version() == 2


def test_error_mapping_without_gpu():
    # argument validation happens before any CUDA call, so it works on a CPU box
    from paper_2505_16864_b200 import _native
    from paper_2505_16864_b200.errors import DomainError, ShapeError, SizeError

    _native.load()
    with pytest.raises(ShapeError):
        _native.call("tcb_curve_build", 0, 4, 4, None, None, None)
    with pytest.raises(SizeError):
        _native.call("tcb_curve_build", 2048, 2048, 2048, 1, 1, None)
    with pytest.raises(DomainError):
        _native.call("tcb_upsample_renoise", 1, None, None, 1, 2, 2, 2, 1, 2, 2, 1, 0.5, 0, 0, 0,
                     None)
    with pytest.raises(DomainError):
        _native.call("tcb_block_pool", 1, None, 7, 0, 0, 1, 1, 1, 1, 1, 1, 0, 1, None, None)
    # carve: unknown dtype, shape errors, too many work items
    # (q, k, v, o, dtype, sh, sn, bits, words, kv_cnt, H, d, m, M_v, M_total, n_valid, n_cond,
    #  beta, work, work_bytes, stream)
    with pytest.raises(DomainError):
        _native.call("tcb_carve_fwd", 1, 1, 1, 1, 9, 128, 128, 1, 1, 1, 1, 128, 128, 1, 1, 1, 0,
                     0.0, 1, 256, None)
    with pytest.raises(ShapeError):
        _native.call("tcb_carve_fwd", None, 1, 1, 1, 1, 128, 128, 1, 1, 1, 1, 128, 128, 1, 1, 1, 0,
                     0.0, 1, 256, None)
    with pytest.raises(ShapeError):  # mask rows narrower than M_total columns
        _native.call("tcb_carve_fwd", 1, 1, 1, 1, 1, 128, 128, 1, 1, 1, 1, 128, 128, 40, 40, 1, 0,
                     0.0, 1, 256, None)
    with pytest.raises(SizeError):
        _native.call("tcb_carve_fwd", 1, 1, 1, 1, 1, 128, 128, 1, 128, 1, 1 << 20, 128, 128, 4096,
                     4096, 1, 0, 0.0, 1, 256, None)
    # selection: M_total beyond the supported range, n_floor < 1
    with pytest.raises(SizeError):
        _native.call("tcb_block_select", 1, 1, 9000, 9000, None, 300, 1, 0.0, 1, 1, 1, None)
    with pytest.raises(DomainError):
        _native.call("tcb_block_select", 1, 1, 4, 4, None, 1, 0, 0.0, 1, 1, 1, None)
    with pytest.raises(DomainError):  # R-free mask: p outside [0, 1)
        _native.call("tcb_block_mask", 1, 4, 1, 1, 4, 4, 128, None, 1, 1, 1.0, 1, 1, 1, 4, None)
    with pytest.raises(SizeError):  # scratch below one row
        _native.call("tcb_block_mask", 1, 4, 1, 1, 4, 4, 128, None, 1, 1, 0.0, 1, 1, 1, 3, None)
    # all C2 heads' scores fit the 256 MB cap; the 8,192-block maximum is chunked under it
    assert _native.query("tcb_block_mask_scratch", 24, 929, 931) == 24 * 929 * 931
    assert 8192 <= _native.query("tcb_block_mask_scratch", 24, 8190, 8192) <= 32 << 20
    # fused neighbours: bad rope sections / strides / patch sizes / grid mismatch
    import ctypes as C
    one = (C.c_void_p * 1)(16)
    rot = (C.c_int * 1)(1)
    with pytest.raises(DomainError):
        _native.call("tcb_rope_permute", C.cast(one, C.c_void_p), 64, 64, C.cast(one, C.c_void_p), 64,
                     64, C.cast(rot, C.c_void_p), 1, 16, 2, 2, 2, 1, 64, 16, 10, 30, 30, None)
    with pytest.raises(ShapeError):
        _native.call("tcb_rope_permute", C.cast(one, C.c_void_p), 63, 64, C.cast(one, C.c_void_p), 64,
                     64, C.cast(rot, C.c_void_p), 1, 16, 2, 2, 2, 1, 64, 16, 0, 32, 32, None)
    with pytest.raises(DomainError):
        _native.call("tcb_unpermute_euler", 1, 1, 1, 2, 2, 2, 0, 1, 1, 1, -0.1, 1, None)
    with pytest.raises(ShapeError):
        _native.call("tcb_curve_positions", 1, 7, 2, 2, 2, 1, None)
    with pytest.raises(ShapeError):
        _native.call("tcb_mask_words_to_packbits", 1, 4, 100, 3, 1, None)


@pytest.fixture(scope="module")
def curve_host(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ missing")
    exe = str(tmp_path_factory.mktemp("cv") / "curve_host")
    subprocess.run([gxx, "-O2", "-std=c++17", "-o", exe,
                    os.path.join(ROOT, "tests", "native", "curve_host.cpp")], check=True)
    return exe


def run_host(exe, dims_list):
    inp = "".join(f"{t} {h} {w}\n" for t, h, w in dims_list)
    out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout
    return [np.array(l.split(), dtype=np.int64) for l in out.strip().split("\n")]


def test_device_curve_math_matches_reference_small(curve_host):
    cases = list(gio.small_curves())
    got = run_host(curve_host, [d for d, _ in cases])
    for (d, fw), g in zip(cases, got):
        assert np.array_equal(g, fw), d


def test_device_curve_math_all_planes_to_40(curve_host):
    dims = [(1, a, b) for a in range(1, 41) for b in range(1, 41)]
    got = run_host(curve_host, dims)
    for d, g in zip(dims, got):
        assert np.array_equal(g, oracle.curve_forward(d)), d


def test_device_curve_math_named_shapes(curve_host):
    g = gio.load("curves.npz")
    import hashlib

    big = [tuple(int(v) for v in d) for d in g["big_dims"]]
    got = run_host(curve_host, big)
    for i, fw in enumerate(got):
        sha = hashlib.sha256(fw.astype("<i8").tobytes()).hexdigest()[:16]
        assert sha == str(g["big_sha"][i]), big[i]


def test_carve_workspace_query_host_only():
    # pure host arithmetic (no GPU): the condition-row split's workspace
    from paper_2505_16864_b200 import _native

    q = lambda *a: _native.query("tcb_carve_workspace_bytes", *a)  # noqa: E731
    assert q(40, 256, 256, 128, 128) == 256               # no text: counter only
    assert q(4, 32, 33, 64, 64) == 256                    # SIMT shapes: counter only
    assert q(24, 929, 931, 128, 128) == 256 + 256 + 24 * 2 * 8 * 128 * 130 * 4   # C2: 8 chunks
    assert q(3, 929, 931, 128, 128) == 256 + 256 + 3 * 2 * 8 * 128 * 130 * 4
    assert q(24, 7000, 7600, 128, 128) == 256             # > 256 MB of partials: unsplit
