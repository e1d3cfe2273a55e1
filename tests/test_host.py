"""CPU-only checks of the product library and its host-side pieces (no GPU needed).

* libhmat_b200.so loads and exports every function include/hmat_b200.h declares;
* the glibc exp/log ports (host build of the same code the device runs) are bit-exact
  against the libm the reference uses;
* without a CUDA device every compute entry point fails loudly (HM_ECUDA) -- there is no
  CPU fallback;
* the synthetic-input generators reproduce the reference's SplitMix64 / Halton streams.
"""
import ctypes
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(REPO, "include", "hmat_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(hm_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol(hm):
    lib = ctypes.CDLL(hm.LIB_PATH)
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(hm.EXPORTED_SYMBOLS) <= set(names)


def test_cpp_facade_header_covers_the_reference_api():
    src = open(os.path.join(REPO, "include", "hmat_b200.hpp")).read()
    for fn in ("setup", "mvp", "cg_solve", "relative_error", "morton_order", "compute_morton_codes", "aca_batched"):
        assert re.search(r"\b" + fn + r"\s*\(", src), fn


def _libm(name):
    libm = ctypes.CDLL("libm.so.6")
    f = getattr(libm, name)
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.c_double]
    return np.frompyfunc(f, 1, 1)


def test_exp_port_host_bitwise(hm):
    rng = np.random.default_rng(11)
    xs = np.concatenate([-rng.uniform(0, 40, 300_000), rng.uniform(-745, 709, 50_000),
                         np.array([0.0, -0.0, 2.0 ** -54, -2.0 ** -55, 512.0, -512.0, -745.2, -1000.0, 1000.0,
                                   np.inf, -np.inf, -708.5, -720.3, 709.78])])
    with np.errstate(over="ignore"):
        want = _libm("exp")(xs).astype(np.float64)
    got = hm.exp_port_host(xs)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_log_port_host_bitwise(hm):
    rng = np.random.default_rng(12)
    xs = np.concatenate([rng.uniform(0, 1, 300_000), rng.uniform(0.9, 1.1, 200_000), np.exp(rng.uniform(-700, 700, 50_000)),
                         np.array([0.0, 1.0, np.inf, 5e-324, 1e-310, 0.9375, 1.064697265625, 0.5, 2.0])])
    with np.errstate(all="ignore"):
        want = _libm("log")(xs).astype(np.float64)
    got = hm.log_port_host(xs)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_no_device_fails_loudly(hm):
    if hm.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    from paper_1708_09707_b200.inputs import uniform_points
    with pytest.raises(hm.HmError) as e:
        hm.setup(uniform_points(256, 2), hm.KernelFunction(), hm.HmatrixConfig(c_leaf=16))
    assert e.value.status == hm.HM_ECUDA
    with pytest.raises(hm.HmError):
        hm.morton_codes(uniform_points(16, 2))


def test_config_validation_errors_are_invalid_argument(hm):
    # validation runs before any device work (hmatrix.cpp:20-26)
    from paper_1708_09707_b200.inputs import uniform_points
    if hm.device_count() > 0:
        pytest.skip("covered by the GPU suite")
    with pytest.raises(hm.HmError):
        hm.setup(uniform_points(32, 2), hm.KernelFunction(), hm.HmatrixConfig(eta=-1.0))


def _splitmix_scalar(seed, count):
    M = (1 << 64) - 1
    state = seed & M
    out = []
    for _ in range(count):
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        out.append(z ^ (z >> 31))
    return out


def test_splitmix_matches_reference_definition():
    from paper_1708_09707_b200.inputs import splitmix64_stream, uniform, symmetric
    for seed in (0, 1, 7, 42, 2 ** 63 + 5):
        assert [int(v) for v in splitmix64_stream(seed, 50)] == _splitmix_scalar(seed, 50)
    u = uniform(42, 1000)
    want = np.array([(v >> 11) * 2.0 ** -53 for v in _splitmix_scalar(42, 1000)])
    assert np.array_equal(u, want)
    assert np.array_equal(symmetric(7, 100), 2.0 * uniform(7, 100) - 1.0)


def test_halton_matches_reference(reference):
    from paper_1708_09707_b200.inputs import halton_points
    for n, d in ((200, 5), (1000, 2), (64, 20)):
        assert np.array_equal(halton_points(n, d).view(np.uint64), reference.halton(n, d).view(np.uint64))


def test_halton_known_values():
    from paper_1708_09707_b200.inputs import halton_points
    p = halton_points(3, 1)
    assert list(p[0]) == [0.5, 0.25, 0.75]
    assert halton_points(2, 2)[1, 1] == pytest.approx(2.0 / 3.0, rel=1e-15)
