"""CPU-side checks of the product library: it loads, exports every symbol the
C ABI header declares, and its host-side arithmetic (reference RNG, coefficient
recipes, parameter selection, μ bound) matches the pinned oracle. No device
compute is called here."""
import math
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "renyi_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(renyi_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(R):
    from paper_2205_07426_b200 import _lib

    lib = _lib.lib()
    declared = header_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signature table must match the header"


def test_no_device_fails_loudly(R):
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except ImportError:
        pass
    with pytest.raises(R.RenyiError) as e:
        R.Context(0)
    assert e.value.kind == "no_device"


def test_rng_bitwise_matches_oracle(R, orc):
    for x in (0, 1, 2**63 + 5, 123456789):
        assert R.mix64(x) == orc.mix64(x)
        assert R.derive_key(x, 77) == orc.derive_key(x, 77)
    for s in ("", "a", "hutchpp-sketch", "term:joint"):
        assert R.hash_name(s) == orc.hash_name(s)
    for kind in ("gaussian", "rademacher"):
        a = R.gaussian_panel(257, 5, 42, "hutchpp-probe", kind)
        b = orc.probe_panel(257, 5, 42, "hutchpp-probe", kind)
        assert np.array_equal(a, b)


def test_coefficients_match_oracle(R, orc):
    for alpha, m in ((1.5, 2), (2.0, 4), (0.5, 30)):
        assert np.array_equal(R.binomial_coeffs(alpha, m), orc.binomial_coeffs(alpha, m))
    for alpha, m, u, v in ((1.5, 40, 0.0, 1.0), (1.01, 60, 0.0, 1.0), (0.5, 15, 0.1, 0.9)):
        assert np.array_equal(R.chebyshev_coeffs(alpha, m, u, v), orc.chebyshev_coeffs(alpha, m, u, v))
    assert R.chebyshev_safeguard(0.1, 0.11) == orc.safeguard(0.1, 0.11)
    assert R.taylor_tail_constant(1.5) == orc.taylor_tail_constant(1.5)
    for spec, ospec in ((R.MatrixFunctionSpec.int_power(3), orc.Spec("int", 3)),
                        (R.MatrixFunctionSpec.taylor(1.3, 12, 0.8), orc.Spec("taylor", 1.3, 12, 0, 0.8)),
                        (R.MatrixFunctionSpec.chebyshev(2.2, 9, 0.1, 0.8), orc.Spec("chebyshev", 2.2, 9, 0.1, 0.8))):
        for lam in (0.1, 0.37, 0.8):
            assert R.scalar_value(spec, lam) == pytest.approx(orc.scalar_value(ospec, lam), rel=1e-14)


def test_chebyshev_node_coeffs_and_method_name(R, orc):  # test_poly.cpp:58-64, entropy.cpp:51-60
    c = R.chebyshev_node_coeffs(lambda x: x, 1, 0.0, 1.0)  # f = lambda on [0, 1]: c0 = 1, c1 = 1/2
    assert c[0] == pytest.approx(1.0, abs=1e-15) and c[1] == pytest.approx(0.5, abs=1e-15)
    for alpha, m, u, v in ((1.5, 40, 0.0, 1.0), (1.01, 60, 0.0, 1.0), (2.5, 30, 0.05, 0.6)):
        np.testing.assert_array_equal(R.chebyshev_node_coeffs(lambda x: x ** alpha, m, u, v),
                                      R.chebyshev_coeffs(alpha, m, u, v))
    with pytest.raises(R.RenyiError):
        R.chebyshev_node_coeffs(math.exp, 0, 0.0, 1.0)
    assert [R.method_name(k) for k in range(5)] == ["exact", "int", "taylor", "chebyshev", "auto"]
    assert R.method_name("chebyshev") == "chebyshev" and R.method_name(9) == "?"


def test_random_stream_bitwise(R, orc):  # rng.hpp:12-36 against the oracle's restatement
    key = orc.derive_key(7, orc.hash_name("X"))
    s = R.RandomStream(key)
    np.testing.assert_array_equal(s.fill_gaussian(500, 3), orc.fill_gaussian(key, 500, 3))
    t = R.RandomStream(11)
    d = t.derive(5)
    assert d.key() == orc.derive_key(11, 5)
    u = [t.next_u64() for _ in range(3)]
    assert u[0] != u[1] and all(0 <= v < 2**64 for v in u)
    assert 0.0 <= t.next_uniform() < 1.0
    g1, g2 = R.RandomStream(3).next_gaussian(), R.RandomStream(3).fill_gaussian(2, 1)[:, 0]
    assert g1 == g2[0]


def test_expected_queries(R):  # test_hutchpp.cpp:74-78
    assert R.expected_queries(R.MatrixFunctionSpec.int_power(2), R.SketchConfig(8)) == 22
    assert R.expected_queries(R.MatrixFunctionSpec.taylor(0.5, 15, 1.0), R.SketchConfig(8)) == 100
    assert R.expected_queries(R.MatrixFunctionSpec.chebyshev(1.5, 15, 0.1, 0.9), R.SketchConfig(16)) == 200


def test_select_params_and_mu_bound(R):  # test_entropy.cpp:157-234
    assert R.select_params(2.0, 0.1, 0.1, R.SpectrumBounds(), 100, "int").s == 20
    p2 = R.select_params(1.5, 0.01, 0.1, R.SpectrumBounds(u=0.001, v=0.1, kappa=100.0), 100, "chebyshev")
    assert p2.m == 100
    p3 = R.select_params(2.0, 0.01, 0.1, R.SpectrumBounds(u=0.0, v=0.5), 1000, "chebyshev")
    assert p3.m == 71
    with pytest.raises(R.RenyiError) as e:
        R.select_params(1.0, 0.1, 0.1, R.SpectrumBounds(), 10, "taylor")
    assert e.value.kind == "alpha_is_one" and e.value.is_usage()
    assert R.mu_bound(0.0, 0.5, 2.0, 10).mu == pytest.approx(0.5, rel=1e-14)
    with pytest.raises(R.RenyiError) as e:
        R.mu_bound(0.05, 0.04, 2.0, 10)
    assert e.value.kind == "invalid_argument"


def test_entropy_from_trace_errors(R):  # test_entropy.cpp:45-55
    assert R.entropy_from_trace(0.38, 2.0) == pytest.approx(-math.log(0.38))
    with pytest.raises(R.RenyiError) as e:
        R.entropy_from_trace(0.0, 2.0)
    assert e.value.kind == "non_positive_trace" and not e.value.is_usage()
    with pytest.raises(R.RenyiError) as e:
        R.entropy_from_trace(1.0, 1.0 + 1e-12)
    assert e.value.kind == "alpha_is_one"


def test_spec_validation(R):  # poly.cpp:60-80
    with pytest.raises(R.RenyiError) as e:
        R.MatrixFunctionSpec.taylor(0.5, 10, 1.5)
    assert e.value.kind == "domain_error"
    with pytest.raises(R.RenyiError):
        R.MatrixFunctionSpec.chebyshev(0.5, 0, 0.0, 1.0)
    with pytest.raises(R.RenyiError):
        R.MatrixFunctionSpec.int_power(0)


def test_cpp_mirror_compiles_links_and_runs(tmp_path):
    """include/renyi_b200.hpp builds against the C ABI with plain g++ (reference toolchain)."""
    import subprocess

    exe = tmp_path / "example_host"
    lib_dir = ROOT / "paper_2205_07426_b200"
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}",
                        str(ROOT / "tests" / "cpp" / "example_host.cpp"), f"-L{lib_dir}", "-lrenyi_b200",
                        f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_mixture_samples_match_oracle(R, orc):
    """mixture_samples (proj/src/simulate.cpp:9-17): one stream, bitwise."""
    x = R.mixture_samples(50, 3, 11, 1.5)
    y = orc.mixture_samples(50, 3, 11, 1.5)
    assert np.array_equal(x, y)


def test_nccl_unique_id_without_gpu(R):
    """The NCCL transport opens libnccl.so.2 at run time; creating the bootstrap id needs no GPU."""
    try:
        uid = R.nccl_unique_id()
    except R.RenyiError as e:  # no libnccl on this host: the error is the NCCL kind, not a crash
        assert e.kind == "nccl_error"
        return
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128 and any(uid)
