"""CPU tests of the boundary and host logic (no GPU): the C-ABI library loads
and exports every symbol include/*.h declares; the partitioner and scheduler
follow the reference's semantics and SPEC examples; GPU entry points fail
loudly (no CPU fallback) when no device is present."""
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2005_08466_b200 import HaoclError, Scheduler, split_ranges, spmv_partition_ranges
from paper_2005_08466_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    syms = set()
    for h in ("hcl_cabi.h", "hcl_host.h", "hcl_datagen.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        syms |= set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(hcl_[a-z_0-9]+)\s*\(", text, re.M))
    return syms


def test_library_exports_every_declared_symbol():
    L = N.lib()
    syms = header_symbols()
    assert len(syms) >= 58
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert syms == set(N.declared_symbols())


def test_gpu_entry_points_fail_loudly_without_a_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2005_08466_b200 import HostContext

    with pytest.raises(HaoclError) as e:
        HostContext()
    assert e.value.name == "precondition"
    assert "no CPU fallback" in str(e.value)


def test_split_ranges_reduces_to_block_range():
    rng = np.random.default_rng(0)
    for _ in range(200):
        total = int(rng.integers(0, 10**12))
        P = int(rng.integers(1, 9))
        w = int(rng.integers(1, 1 << 20))
        # proj/src/bench.cpp:31-33
        assert split_ranges(total, [w] * P) == [total * i // P for i in range(P + 1)]


def test_split_ranges_weighted_matches_oracle_and_is_proportional():
    rng = np.random.default_rng(1)
    for _ in range(100):
        P = int(rng.integers(1, 9))
        w = [int(x) for x in rng.integers(1, 1000, P)]
        total = int(rng.integers(0, 10**9))
        b = split_ranges(total, w)
        assert b == O.weighted_ranges(total, w).tolist()
        assert b[0] == 0 and b[-1] == total and all(x <= y for x, y in zip(b, b[1:]))
        for i in range(P):  # each share within one row of exact proportion
            assert abs((b[i + 1] - b[i]) - total * w[i] / sum(w)) <= 1.0 + 1e-9 * total


def test_spmv_partition_matches_reference(golden):
    for key, case in golden["spmv_partition"].items():
        if not key.startswith("skew"):
            continue
        rp = np.array(case["row_ptr"], np.int64)
        P = int(key.rsplit("_P", 1)[1])
        if case["rc"] != 0:
            with pytest.raises(HaoclError) as e:
                spmv_partition_ranges(rp, P)
            assert e.value.code == case["rc"]  # argument (9)
        else:
            assert spmv_partition_ranges(rp, P).tolist() == case["ranges"], key


def test_spmv_partition_weighted_matches_oracle():
    rng = np.random.default_rng(5)
    for _ in range(100):
        rows = int(rng.integers(2, 300))
        rp = np.concatenate([[0], np.cumsum(rng.integers(0, 40, rows) ** 2)]).astype(np.int64)
        P = int(rng.integers(1, min(rows, 8) + 1))
        w = [int(x) for x in rng.integers(1, 100, P)]
        assert (spmv_partition_ranges(rp, P, w) == O.spmv_partition_ranges(rp, P, w)).all()
        assert (spmv_partition_ranges(rp, P) == O.spmv_partition_ranges(rp, P)).all()


def test_spmv_partition_greedy_bound():
    # max part nnz <= ceil(nnz/P) + max_row_nnz
    rng = np.random.default_rng(9)
    for _ in range(200):
        rows = int(rng.integers(1, 200))
        lens = rng.integers(0, 60, rows) ** int(rng.integers(1, 3))
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        P = int(rng.integers(1, rows + 1))
        r = spmv_partition_ranges(rp, P)
        nnz = int(rp[-1])
        assert r[0] == 0 and r[-1] == rows and (np.diff(r) >= 1).all()
        for p in range(P):
            assert rp[r[p + 1]] - rp[r[p]] <= -(-nnz // P) + int(lens.max(initial=0))


# ---- scheduler: SPEC.md scheduler module examples -------------------------


def test_round_robin_cycles_and_balances():
    s = Scheduler([(0, 1.0), (1, 1.0), (2, 1.0)])
    assert [s.schedule("vecadd", "round_robin") for _ in range(7)] == [0, 1, 2, 0, 1, 2, 0]
    s4 = Scheduler([(g, 1.0) for g in range(4)])
    picks = [s4.schedule("matmul", "round_robin") for _ in range(12)]
    assert [picks.count(g) for g in range(4)] == [3, 3, 3, 3]


def test_cost_model_published_formula():
    s = Scheduler([(0, 1.0), (1, 8.0)])
    assert s.modeled_cost(0, "matmul", 1e9) == pytest.approx(1.0)
    assert s.modeled_cost(1, "matmul", 1e9) == pytest.approx(0.125)
    assert s.schedule("matmul", "cost_model", work_units=1e9) == 1
    # tie -> smaller id; data term charged when not resident
    t = Scheduler([(0, 2.0), (1, 2.0), (2, 2.0)])
    assert t.schedule("knn", "cost_model", work_units=5e8) == 0
    assert t.modeled_cost(0, "knn", 1e9, in_bytes=10**8, resident=False) == pytest.approx(0.5 + 1.0)
    t.note_resident(77, [2])
    assert t.schedule("knn", "cost_model", work_units=1e9, in_bytes=10**9, buffers=[77]) == 2


def test_cost_model_invariances():
    rng = np.random.default_rng(2)
    for _ in range(30):
        rates = [float(x) for x in rng.uniform(0.1, 10, 4)]
        base = Scheduler(list(enumerate(rates))).schedule("m", "cost_model", work_units=1e9)
        scaled = Scheduler([(i, r * 7.5) for i, r in enumerate(rates)]).schedule("m", "cost_model", work_units=1e9)
        assert base == scaled
        boosted = list(rates)
        boosted[base] *= 2.0
        assert Scheduler(list(enumerate(boosted))).schedule("m", "cost_model", work_units=1e9) == base


def test_ema_profile_recurrence_and_errors():
    s = Scheduler([(0, 1.0)])
    s.record_profile(0, "matmul", 1e6, 1.0)
    assert s.rate(0, "matmul") == 1e6
    s.record_profile(0, "matmul", 2e6, 1.0)
    assert abs(s.rate(0, "matmul") - 1.3e6) < 1e-12 * 1.3e6
    with pytest.raises(HaoclError) as e:
        s.record_profile(0, "matmul", 1.0, 0.0)
    assert e.value.name == "precondition"
    with pytest.raises(HaoclError) as e:
        s.record_profile(5, "matmul", 1.0, 1.0)
    assert e.value.name == "unknown_device"


def test_policy_registry_and_static_map():
    s = Scheduler([(0, 1.0), (1, 1.0)], kernel_map={"spmv_partition": 1})
    s.register_fixed_policy("mine", 0)
    assert all(s.schedule("vecadd", "mine") == 0 for _ in range(5))
    with pytest.raises(HaoclError) as e:
        s.register_fixed_policy("round_robin", 0)
    assert e.value.name == "registration"
    assert s.schedule("spmv_partition", "static_map") == 1
    with pytest.raises(HaoclError) as e:
        s.schedule("spmv_compute", "static_map")
    assert e.value.name == "mapping"
    with pytest.raises(HaoclError) as e:
        s.schedule("vecadd", None, device=9)
    assert e.value.name == "unknown_device"
    assert s.schedule("vecadd", None, device=1) == 1  # user_directed honours explicit placement
    with pytest.raises(HaoclError) as e:
        s.schedule("vecadd", "nosuch")
    assert e.value.name == "policy"


def test_partition_weights_follow_measured_rates():
    s = Scheduler([(0, 1.0), (1, 1.0), (2, 1.0)])
    w = s.partition_weights("gemm_bf16", [0, 1, 2])
    assert w[0] == w[1] == w[2]
    s.record_profile(0, "gemm_bf16", 3e12, 1.0)
    s.record_profile(1, "gemm_bf16", 1e12, 1.0)
    s.record_profile(2, "gemm_bf16", 2e12, 1.0)
    w = s.partition_weights("gemm_bf16", [0, 1, 2])
    assert w[0] == 1 << 20 and abs(w[1] / w[0] - 1 / 3) < 1e-5 and abs(w[2] / w[0] - 2 / 3) < 1e-5
    b = split_ranges(16384, w)
    assert b[1] - b[0] == pytest.approx(16384 / 2, abs=1)


def test_product_datagen_matches_oracle_streams():
    from paper_2005_08466_b200 import datagen as G

    assert (G.gen_doubles(10**5, 42) == O.gen_doubles(10**5, 42)).all()
    full = O.gen_doubles(300000, 43)
    assert (G.gen_doubles(1000, 43, first=123456) == full[123456:124456]).all()  # any sub-range
    assert (G.gen_bf16(300000, 42) == O.gen_bf16(300000, 42)).all()
    assert (G.gen_f32(1000, 9) == O.gen_doubles(1000, 9).astype(np.float32)).all()
    s, d = G.gen_rmat_edges(12, 70000, 42, first=5)
    s2, d2 = O.rmat_edges(12, 5, 70000, 42)
    assert (s == s2).all() and (d == d2).all()
    assert (G.gen_kmeans_points(70000, 8, 16, 42, first=3) == O.kmeans_points(42, 3, 70000, 8, 16)).all()


def test_scheduler_profiles_persist(tmp_path):
    """EMA profiles survive a save/load round trip exactly (§8(f) 2) and drive
    the same partition weights; devices the new run lacks are skipped."""
    from paper_2005_08466_b200 import HaoclError, Scheduler

    s = Scheduler([(1, 1.0), (2, 1.0), (3, 1.0)])
    for sec in (0.010, 0.012, 0.011):
        s.record_profile(1, "conv3x3", 1e9, sec)
        s.record_profile(2, "conv3x3", 1e9, sec * 2.1)
    s.record_profile(3, "gemm_bf16", 5e12, 0.0037)
    path = str(tmp_path / "profiles.tsv")
    s.save_profiles(path)
    t = Scheduler([(1, 1.0), (2, 1.0)])
    assert t.load_profiles(path) == 2  # device 3 is not in this run
    assert t.rate(1, "conv3x3") == s.rate(1, "conv3x3") and t.rate(2, "conv3x3") == s.rate(2, "conv3x3")
    assert t.partition_weights("conv3x3", [1, 2]) == s.partition_weights("conv3x3", [1, 2])
    bad = tmp_path / "bad.tsv"
    bad.write_text("1 conv3x3 5\n")
    with pytest.raises(HaoclError) as e:
        t.load_profiles(str(bad))
    assert e.value.name == "parse"
