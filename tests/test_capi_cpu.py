"""CPU-only checks of the C-ABI boundary: the product library loads, exports
every entry point include/*.h declares, keeps the reference's host-side
semantics (spec validation messages, Theorem 2.1), never touches the oracle,
and fails loudly (no CPU fallback) when asked to compute without a GPU."""
import ctypes as C
import glob
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from helpers import sweep_specs

import paper_2411_19419_b200 as sp


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(spconv_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 16
    lib = C.CDLL(sp.library_path)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_and_oracle_free():
    so = sp.library_path
    needed = subprocess.run(["readelf", "-d", so], capture_output=True, text=True).stdout
    assert "oracle" not in needed and "spconv_ref" not in needed
    syms = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
    assert "orc_" not in syms and "ref_" not in syms.replace("spconv_", "")
    sass = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in sass


def test_abi_version():
    assert sp.lib.spconv_abi_version() >= 100


def test_spec_validation_messages(ref=None):
    with pytest.raises(ValueError, match=r"^ConvSpec: need m,n,k,s >= 1 and p >= 0, got "
                                         r"\(m=0, n=3, k=1, s=1, p=0\)$"):
        sp.ConvSpec(0, 3, 1, 1, 0)
    with pytest.raises(ValueError, match=r"^ConvSpec: kernel larger than padded input, "
                                         r"\(m=3, n=3, k=6, s=1, p=1\)$"):
        sp.ConvSpec(3, 3, 6, 1, 1)
    with pytest.raises(ValueError, match="Kernel: expected 4 values, got 1"):
        sp.Kernel(2, [1.0])


def test_spec_messages_match_reference(ref):
    from oracle import RefError
    for args in [(0, 3, 1, 1, 0), (3, 3, 1, 0, 0), (3, 3, 1, 1, -1), (3, 3, 6, 1, 1), (2, 9, 5, 1, 1)]:
        with pytest.raises(RefError) as e:
            ref.spec_check(*args)
        with pytest.raises(ValueError) as g:
            sp.ConvSpec(*args)
        assert str(g.value) == str(e.value)


def test_nnz_bound_matches_oracle(orc):
    for spec in sweep_specs(9):
        assert sp.nnz_bound(sp.ConvSpec(*spec)) == orc.nnz_bound(*spec)
    for spec in [(64, 64, 3, 1, 1), (512, 512, 5, 2, 2), (1024, 1024, 3, 1, 1), (4096, 4096, 7, 2, 3),
                 (257, 193, 11, 1, 10)]:
        assert sp.nnz_bound(sp.ConvSpec(*spec)) == orc.nnz_bound(*spec)
    assert sp.nnz_bound(sp.ConvSpec(4096, 4096, 7, 2, 3)) == 205348900


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="cuda|CUDA"):
        sp.build_transform(sp.Kernel(3, np.ones(9)), sp.ConvSpec(8, 8, 3, 1, 1))


def test_dropin_headers_compile():
    """The drop-in C++ headers compile standalone (-fsyntax-only)."""
    src = '#include "spconv/spconv.hpp"\nint main(){ spconv::ConvSpec s(3,3,3,1,1); return (int)s.m_out(); }\n'
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-I",
                        os.path.join(ROOT, "include"), "-x", "c++", "-"], input=src, text=True,
                       capture_output=True)
    assert r.returncode == 0, r.stderr


def test_int32_range_rejected_before_any_device_work():
    """Geometries past the int32 device index range (m*n or nnz >= 2^31) are
    rejected with std::invalid_argument semantics before the device is touched
    (so this runs without a GPU)."""
    with pytest.raises(ValueError, match="exceeds the int32 device index range"):
        sp.build_transform(sp.Kernel(1, [1.0]), sp.ConvSpec(46341, 46341, 1, 1, 0))
    with pytest.raises(ValueError, match=r"nnz \d+ exceeds the int32 device index range"):
        sp.build_transform(sp.Kernel(11, np.ones(121)), sp.ConvSpec(20000, 20000, 11, 1, 5))
    with pytest.raises(ValueError, match="layout must be 0"):
        sp.build_transform(sp.Kernel(3, np.ones(9)), sp.ConvSpec(8, 8, 3, 1, 1), layout=2)
    with pytest.raises(ValueError, match="unknown layout 'coo'"):
        sp.layout_from_name("coo")
    # double taps fp32 cannot hold (spconv_build_transform_f64): the same checks, same order
    taps = np.full(9, 0.1)
    with pytest.raises(ValueError, match="layout must be 0"):
        sp.build_transform(sp.Kernel(3, taps), sp.ConvSpec(8, 8, 3, 1, 1), layout=2)
    with pytest.raises(ValueError, match=r"nnz \d+ exceeds the int32 device index range"):
        sp.build_transform(sp.Kernel(3, taps), sp.ConvSpec(20000, 20000, 3, 1, 1))
    with pytest.raises(ValueError, match="kernel larger than padded input"):
        sp.build_transform(sp.Kernel(3, taps), sp.ConvSpec(1, 1, 3, 1, 0))


def test_rng_matches_reference_known_answers(golden, orc):
    """The library's seeded generator (inc/rng.hpp, behind the drop-in rng.hpp)
    reproduces the reference's known answers and the oracle's streams."""
    js, _ = golden
    assert str(sp.lib.spconv_derive_seed(42, 0)) == js["derive_seed_42_0"]
    out = np.empty(3)
    sp._check(sp.lib.spconv_random_normal(42, 3, out.ctypes.data))
    assert out.tolist() == js["normal_42_first3"]
    for seed in (1, 7, orc.derive_seed(42, 5)):
        assert sp.lib.spconv_derive_seed(seed, 9) == orc.derive_seed(seed, 9)
        got = np.empty(1001)
        sp._check(sp.lib.spconv_random_normal(seed, 1001, got.ctypes.data))
        assert np.array_equal(got.view(np.uint64), orc.random_normal(seed, 1001).view(np.uint64))


def test_coo_checks_before_any_device_work():
    """spconv_matrix_from_coo: Triplets' dimension and range checks, same
    messages, raised on the host (runs without a GPU)."""
    with pytest.raises(ValueError, match=r"^Triplets: dimensions must be at least 1x1, got 0x3$"):
        sp.compile_triplets(0, 3, [], [], [])
    with pytest.raises(ValueError, match=r"^Triplets: entry \(2, 5\) outside 3x5$"):
        sp.compile_triplets(3, 5, [0, 2], [1, 5], [1.0, 2.0])
    with pytest.raises(ValueError, match="layout must be 0"):
        sp.compile_triplets(3, 5, [0], [1], [1.0], layout=3)


def test_path_options_roundtrip_and_errors():
    """spconv_set_option / spconv_get_option: symbolic and integer values round
    trip, unknown names and values are status 1, and the library's sources read
    no environment variables (the options replace them)."""
    with sp.options(path="tiled", fused="1", build="persist", spec_skew=-3):
        assert sp.get_option("path") == "tiled"
        assert sp.get_option("fused") == "1"
        assert sp.get_option("build") == "persist"
        assert sp.get_option("spec_skew") == "-3"
    assert sp.get_option("path") == "auto" and sp.get_option("spec_skew") == "0"
    with pytest.raises(ValueError, match="unknown option"):
        sp.set_option("nope", "1")
    with pytest.raises(ValueError, match="bad value"):
        sp.set_option("path", "warp")
    with pytest.raises(ValueError, match="integer"):
        sp.set_option("spec_skew", "x")
    for src in glob.glob(os.path.join(ROOT, "paper_2411_19419_b200", "csrc", "*.cu")):
        assert "getenv" not in open(src).read(), src


def test_group_argument_checks_without_a_device():
    """The grouped entries validate their arguments before any device work:
    a negative count, null arrays, and the empty group (a no-op)."""
    L = sp.lib
    for fn in (L.spconv_spmv_group, L.spconv_spmv_group_f64):
        assert fn(None, -1, None, None, None) == 1
        assert "negative count" in L.spconv_last_error().decode()
        assert fn(None, 2, None, None, None) == 1
        assert "null array" in L.spconv_last_error().decode()
        assert fn(None, 0, None, None, None) == 0
    for fn in (L.spconv_convolve_host_group, L.spconv_convolve_host_group_f64):
        assert fn(None, -3, None, None) == 1
        assert fn(None, 0, None, None) == 0
    with pytest.raises(ValueError, match="one vector per transform"):
        sp.spmv_group([], [np.zeros(3)])
    with pytest.raises(ValueError, match="one image per transform"):
        sp.convolve_group([], [np.zeros(3)])
