"""CPU-side checks of the C-ABI library: it loads, exports every declared symbol, validates
arguments on the host exactly like the reference, and refuses to compute without a GPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparsekit_b200.h")


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_2605_08575_b200 import _lib
    return _lib


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(skb_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_are_exported(lib):
    names = declared_functions()
    assert len(names) >= 15
    L = lib.load()
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/sparsekit_b200.h but not exported"
    assert sorted(lib.EXPORTS) == names
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True)
    exported = set(re.findall(r" T (skb_\w+)", out.stdout))
    assert exported == set(names)
    assert L.skb_abi_version() == 3


def test_library_does_not_link_the_oracle_or_torch(lib):
    out = subprocess.run(["ldd", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "torch" not in out and "sparsekit_ref" not in out


def test_struct_layouts_match_header(lib):
    assert C.sizeof(lib.SkbConfig) == 32
    assert C.sizeof(lib.SkbReport) == 72
    assert C.sizeof(lib.SkbForwardArgs) == 16 + 16 + 8 * 14 + 8 + 8  # + tau, reserved2, slot_n_off (ABI 3)


def test_config_validate_matches_reference_messages(lib):
    # proj/src/model.cpp:113-127
    L = lib.load()
    cases = [
        ((0, 1, 1, 1, 0, 0, 1, 64), "n_experts must be >= 1"),
        ((4, 0, 1, 1, 0, 0, 1, 64), "top_k must satisfy 1 <= K <= E, got K=0 E=4"),
        ((4, 5, 1, 1, 0, 0, 1, 64), "top_k must satisfy 1 <= K <= E, got K=5 E=4"),
        ((4, 2, 0, 1, 0, 0, 1, 64), "d_model must be >= 1"),
        ((4, 2, 8, 0, 0, 0, 1, 64), "d_ffn must be >= 1"),
        ((4, 2, 8, 8, 0, -1, 1, 64), "d_shared must be >= 0"),
        ((4, 2, 8, 8, 1, 0, 1, 64), "has_shared must match d_shared > 0"),
        ((4, 2, 8, 8, 0, 3, 1, 64), "has_shared must match d_shared > 0"),
        ((4, 2, 8, 8, 0, 0, 1, 0), "align_block must be >= 1"),
    ]
    for fields, msg in cases:
        cfg = lib.SkbConfig(*fields)
        assert L.skb_config_validate(C.byref(cfg)) == lib.SKB_ECONFIG
        assert L.skb_last_error().decode() == msg
    ok = lib.SkbConfig(4, 2, 8, 8, 1, 3, 0, 1)
    assert L.skb_config_validate(C.byref(ok)) == lib.SKB_OK


def test_n_off_matches_oracle(lib, oracle):
    L = lib.load()
    out = C.c_int32()
    for n in list(range(0, 70)) + [511, 512, 1024, 2880, 8192]:
        for s in (0.0, 0.1, 0.25, 0.5, 0.75, 0.9, 0.999, 1.0):
            assert L.skb_n_off(s, n, C.byref(out)) == 0
            assert out.value == oracle.n_off(s, n)
    assert L.skb_n_off(1.5, 8, C.byref(out)) == lib.SKB_ECONFIG
    assert L.skb_n_off(float("nan"), 8, C.byref(out)) == lib.SKB_ECONFIG


def test_argument_validation_precedes_device_work(lib):
    L = lib.load()
    logits = np.zeros((2, 4), np.float32)
    ids = np.zeros((2, 5), np.int32)
    w = np.zeros((2, 5), np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    assert L.skb_route(p(logits), 0, 4, 1, 1, p(ids), p(w)) == lib.SKB_ESHAPE
    assert L.skb_route(p(logits), 2, 4, 5, 1, p(ids), p(w)) == lib.SKB_ECONFIG
    assert b"outside [1, 4]" in L.skb_last_error()
    bad = np.array([[0, 9]], np.int32)
    n1, n2 = C.c_int32(), C.c_int32()
    assert L.skb_align_dispatch(p(bad), 1, 2, 4, 4, p(ids), p(ids), C.byref(n1), C.byref(n2)) == lib.SKB_EINDEX
    assert L.skb_align_dispatch(p(bad), 1, 2, 4, 0, p(ids), p(ids), C.byref(n1), C.byref(n2)) == lib.SKB_ECONFIG


def test_no_cpu_fallback(lib):
    """Without a CUDA device every compute entry point fails loudly with SKB_ECUDA."""
    L = lib.load()
    if L.skb_device_count() > 0:
        pytest.skip("a GPU is present; the refusal path is exercised on CPU-only hosts")
    cfg = lib.SkbConfig(4, 2, 8, 8, 0, 0, 1, 64)
    h = C.c_void_p()
    assert L.skb_layer_create_synthetic(C.byref(cfg), 1, C.c_float(0.1), 0, C.byref(h)) == lib.SKB_ECUDA
    assert b"no CUDA device" in L.skb_last_error()
    logits = np.zeros((2, 4), np.float32)
    ids = np.zeros((2, 2), np.int32)
    w = np.zeros((2, 2), np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    assert L.skb_route(p(logits), 2, 4, 2, 1, p(ids), p(w)) == lib.SKB_ECUDA
    hrow = np.zeros((1, 8), np.float32)
    mask = np.zeros((1, 8), np.uint8)
    assert L.skb_topk_mask(p(hrow), 1, 8, 0.5, p(mask)) == lib.SKB_ECUDA


def test_python_mirror_validates_like_the_reference():
    import paper_2605_08575_b200 as skb
    with pytest.raises(skb.ConfigError):
        skb.SparsityLevel(-0.1)
    with pytest.raises(skb.ConfigError):
        skb.MoEConfig(4, 9, 8, 8).validate()
    skb.MoEConfig(4, 2, 8, 8).validate()
    assert skb.n_off(0.5, 1024) == 512 and skb.n_off(0.9, 1024) == 922


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2605_08575_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in text and "moe_oracle" not in text and "libsparsekit_ref" not in text, f


# ---------------------------------------------------------------------------------------------
# C++ facade (include/sparsekit_b200.hpp)
# ---------------------------------------------------------------------------------------------
FACADE_SRC = os.path.join(ROOT, "tests", "cpp", "facade_check.cpp")


def build_facade_check(lib, out):
    libdir = os.path.dirname(lib.LIB_PATH)
    cmd = ["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), FACADE_SRC, "-o", out,
           "-L", libdir, "-lsparsekit_b200", f"-Wl,-rpath,{libdir}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return out


def test_cpp_facade_builds_against_stand_in_types(lib, tmp_path):
    exe = build_facade_check(lib, str(tmp_path / "facade_check"))
    res = subprocess.run([exe], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "facade" in res.stdout


@pytest.mark.skipif(not os.path.exists("/root/reference/proj/include/sparsekit/engine.hpp"),
                    reason="reference headers not present (GPU box)")
def test_cpp_facade_compiles_against_the_reference_headers():
    """Drop-in proof: with the reference tree on the include path the facade takes its value and
    exception types from the reference's own headers, and the same client code compiles."""
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
           "-I", "/root/reference/proj/include", FACADE_SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


# ---------------------------------------------------------------------------------------------
# host-side pieces of the dense/sparse switch (no device needed)
# ---------------------------------------------------------------------------------------------
def test_generate_tokens_matches_the_oracle_bit_for_bit(lib):
    """skb_generate_tokens vs the oracle's restatement of model.cpp:168-178 / rng.hpp:42-55."""
    from oracle.pyoracle import Oracle
    ork = Oracle.get()
    L = lib.load()
    for batch, d, seed in [(1, 1, 0), (3, 7, 2), (4, 96, 9), (16, 2048, 3), (5, 33, (1 << 64) - 1)]:
        out = np.empty((batch, d), np.float32)
        assert L.skb_generate_tokens(batch, d, seed, out.ctypes.data) == 0
        ref = ork.generate_tokens(batch, d, seed)
        assert out.tobytes() == np.asarray(ref, np.float32).tobytes()
    assert L.skb_generate_tokens(0, 8, 1, None) == 2  # ConfigError, model.cpp:169-171
    assert b"batch >= 1" in L.skb_last_error()


# ---------------------------------------------------------------------------------------------
# neuron budgets: host arithmetic of budget.cpp (KATs of proj/tests/budget_test.cpp:16-137)
# ---------------------------------------------------------------------------------------------
def test_group_experts_and_allocate_budget_hand_cases(lib):
    import paper_2605_08575_b200 as skb
    g = skb.group_experts([0.3, 0.25, 0.2, 0.15, 0.07, 0.03])
    assert (g.g0, g.g1, g.g2) == ([0, 1], [2, 3], [4, 5])
    g7 = skb.group_experts([0.7, 0.6, 0.5, 0.4, 0.3, 0.2, 0.1])
    assert (len(g7.g0), len(g7.g1), len(g7.g2)) == (2, 2, 3)
    g1 = skb.group_experts([1.0])
    assert (g1.g0, g1.g1, g1.g2) == ([], [], [0])
    gt = skb.group_experts([0.2, 0.5, 0.2, 0.1, 0.5, 0.1])  # ties toward the lower slot
    assert (gt.g0, gt.g1, gt.g2) == ([1, 4], [0, 2], [3, 5])
    with pytest.raises(skb.ConfigError):
        skb.group_experts([])

    counts = skb.allocate_budget(6, 8, 0.5, g, skb.BudgetRatios(3.0, 2.0, 1.0))
    assert counts == [6, 6, 4, 4, 2, 2] and sum(counts) == 24
    ge = skb.group_experts([0.4, 0.3, 0.2, 0.06, 0.03, 0.01])
    assert skb.allocate_budget(6, 16, 0.25, ge, skb.BudgetRatios()) == [4] * 6
    g3 = skb.group_experts([0.5, 0.3, 0.2])
    assert skb.allocate_budget(3, 8, 0.0, g3, skb.BudgetRatios(3.0, 2.0, 1.0)) == [0, 0, 0]
    for bad in (skb.BudgetRatios(0.0, 0.0, 0.0), skb.BudgetRatios(-1.0, 1.0, 1.0)):
        with pytest.raises(skb.ConfigError):
            skb.allocate_budget(3, 8, 0.5, g3, bad)
    with pytest.raises(skb.ConfigError):  # K = 1: all mass must sit on g2
        skb.allocate_budget(1, 8, 0.5, g1, skb.BudgetRatios(3.0, 2.0, 0.0))
    assert skb.allocate_budget(1, 8, 0.5, g1, skb.BudgetRatios(3.0, 2.0, 1.0)) == [4]
    with pytest.raises(skb.ConfigError):
        skb.allocate_budget(3, 8, 1.5, g3, skb.BudgetRatios())
    with pytest.raises(skb.ConfigError):  # groups must partition the slots
        skb.allocate_budget(3, 8, 0.5, skb.ExpertGroups([0], [1], []), skb.BudgetRatios())
    with pytest.raises(IndexError):
        skb.allocate_budget(3, 8, 0.5, skb.ExpertGroups([0], [1], [7]), skb.BudgetRatios())

    # rounding slack and clamping bounds, monotone in r0 (budget_test.cpp:90-137)
    rng = np.random.default_rng(53)
    for _ in range(200):
        k, n = int(rng.integers(1, 9)), int(rng.integers(1, 65))
        s_act = float(rng.random())
        r = skb.BudgetRatios(rng.random() * 4, rng.random() * 4, rng.random() * 4 + 0.01)
        groups = skb.group_experts(rng.random(k).astype(np.float32) + 0.01)
        c = skb.allocate_budget(k, n, s_act, groups, r)
        assert all(0 <= v <= n for v in c) and sum(c) <= k * n
        denom = r.r0 * len(groups.g0) + r.r1 * len(groups.g1) + r.r2 * len(groups.g2)
        shares = [s_act * k * n * q / denom for q in (r.r0, r.r1, r.r2)]
        if all(0.0 <= sh <= n for sh in shares):
            assert abs(sum(c) - s_act * k * n) <= k / 2.0 + 3.0
    gm = skb.group_experts([0.5, 0.25, 0.13, 0.07, 0.03, 0.02])
    seq = [skb.allocate_budget(6, 32, 0.4, gm, skb.BudgetRatios(r0, 1.0, 1.0))[gm.g0[0]]
           for r0 in (0.5, 1.0, 2.0, 4.0, 8.0)]
    assert seq == sorted(seq)
