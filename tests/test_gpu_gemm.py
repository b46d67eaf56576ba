"""GPU parity of the tensor-core GEMM (configs C1/C2) against the fp64 oracle
of the same rounded inputs, with the normwise tolerance of SURVEY.md §8(c):
err_ij = |C - C64|_ij / (|A| |B|)_ij. Tolerances (stated here, per path):
  bf16 inputs, fp32 out  : 2^-12   (exact bf16 products, fp32 tensor-core
                                    accumulation; tighter than §8(c)'s 2^-10)
  bf16 inputs, bf16 out  : |C - C64| <= 2^-10 (1 + 2^-8) (|A||B|) + 2^-8 |C64|
                           (§8(c)'s 2^-10 product bound, then one bf16 rounding
                           of the fp32 result: 8-bit significand, unit roundoff 2^-8)
  tf32 (fp32 inputs)     : 2^-10   (1xTF32 products)
  fp32 SIMT (gemm_f32)   : 2^-20   (the fp32-exact path of §8(c): exact fp32
                                    products, k-ascending FFMA chains)
  3xTF32 (gemm_f32x3)    : 2^-16   (the FAST fp32 path, not fp32-exact: exact
                                    split products, but the tensor core's fp32
                                    accumulation truncates per MMA; measured
                                    2^-18.8 at K=1024 unsplit, 2^-17.1 at
                                    K=16384) -- and 2^-20 at C1 (1024^3), where
                                    the default K split into 4 slices summed
                                    in order (2^-20.8 measured) applies
plus bit-identity of C across partitions P in {1,2,4} (P-invariance). The
full-size C2 samples are checked against the reference library's own
kernels::execute("matmul") (oracle/_ref, proj/src/kernels.cpp:96-119)."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2005_08466_b200 import HaoclError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def queues(ctx):
    qs = [ctx.create_queue(g) for g in ctx.get_device_ids()[:4]]
    yield qs
    for q in qs:
        ctx.release(q)


def gemm(ctx, queues, kernel, a, b, m, k, n, out_f32=True, P=1, weights=None):
    prog = ctx.create_program("b200")
    kh = ctx.create_kernel(prog, kernel)
    es_out = 4 if out_f32 else 2
    ba, bb, bc = ctx.create_buffer(a.nbytes), ctx.create_buffer(b.nbytes), ctx.create_buffer(m * n * es_out)
    ctx.enqueue_write_buffer(queues[0], ba, a)
    ctx.enqueue_write_buffer(queues[0], bb, b)
    args = [ba, bb, bc, m, k, n] + ([int(out_f32)] if kernel == "gemm_bf16" else [])
    for i, v in enumerate(args):
        ctx.set_kernel_arg(kh, i, v)
    if P == 1:
        ctx.enqueue_ndrange_kernel(queues[0], kh, (m, n, 1), 2)
    else:
        ctx.enqueue_ndrange_partitioned(kh, (m, n, 1), 2, queues[:P], weights)
    for q in queues[:P]:
        ctx.finish(q)
    raw = ctx.enqueue_read_buffer(queues[0], bc)
    for x in (ba, bb, bc):
        ctx.release(x)
    ctx.release(kh)
    ctx.release(prog)
    if out_f32:
        return raw.view(np.float32).reshape(m, n)
    return O.bf16_to_f32(raw.view(np.uint16)).reshape(m, n)


def assert_bf16_out(c, a64, b64):
    """bf16 output: the 2^-10 bf16-product bound of SURVEY.md §8(c), then one
    bf16 rounding of the fp32 result (8-bit significand: unit roundoff 2^-8)."""
    ref = a64 @ b64
    scale = np.abs(a64) @ np.abs(b64)
    assert (np.abs(c.astype(np.float64) - ref) <= 2.0**-10 * (1 + 2.0**-8) * scale + 2.0**-8 * np.abs(ref)).all()


def normwise_err(c, a64, b64):
    ref = a64 @ b64
    scale = np.abs(a64) @ np.abs(b64)
    return float((np.abs(c.astype(np.float64) - ref) / np.maximum(scale, 1e-300)).max())


SHAPES = [(256, 256, 64), (512, 512, 512), (1024, 1024, 1024), (300, 200, 136), (128, 264, 1000), (777, 520, 72)]


@pytest.mark.parametrize("m,n,k", SHAPES)
@pytest.mark.parametrize("variant", ["cg2_mn", "cg1_mn", "cg2_kmajor", "cg1_kmajor"])
def test_gemm_bf16_fp32out(ctx, queues, m, n, k, variant, monkeypatch):
    monkeypatch.setenv("HCL_GEMM_CG", "2" if variant.startswith("cg2") else "1")
    monkeypatch.setenv("HCL_GEMM_B_KMAJOR", "1" if variant.endswith("kmajor") else "0")
    a = O.gen_bf16(m * k, 42)
    b = O.gen_bf16(k * n, 43)
    c = gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=True)
    a64 = O.bf16_to_f32(a).astype(np.float64).reshape(m, k)
    b64 = O.bf16_to_f32(b).astype(np.float64).reshape(k, n)
    assert normwise_err(c, a64, b64) <= 2.0**-12


@pytest.mark.parametrize("m,n,k", SHAPES[:4])
def test_gemm_bf16_bf16out(ctx, queues, m, n, k):
    a = O.gen_bf16(m * k, 42)
    b = O.gen_bf16(k * n, 43)
    c = gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=False)
    a64 = O.bf16_to_f32(a).astype(np.float64).reshape(m, k)
    b64 = O.bf16_to_f32(b).astype(np.float64).reshape(k, n)
    assert_bf16_out(c, a64, b64)


@pytest.mark.parametrize("P,weights", [(2, None), (4, None), (4, [3, 1, 2, 2])])
def test_gemm_bf16_partition_invariance(ctx, queues, P, weights):
    m, n, k = 1024, 768, 512
    a = O.gen_bf16(m * k, 42)
    b = O.gen_bf16(k * n, 43)
    whole = gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=True)
    part = gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=True, P=P, weights=weights)
    assert whole.tobytes() == part.tobytes()


@pytest.mark.parametrize("m,n,k", [(256, 256, 64), (300, 200, 136), (777, 520, 72), (1024, 1024, 1024)])
@pytest.mark.parametrize("shape", ["0", "1", "2", "3"])  # (CG, BN) = (2,256) (1,256) (2,128) (1,64)
def test_gemm_tile_shapes(ctx, queues, m, n, k, shape, monkeypatch):
    monkeypatch.setenv("HCL_GEMM_SHAPE", shape)
    a = O.gen_bf16(m * k, 42)
    b = O.gen_bf16(k * n, 43)
    c = gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=True)
    a64 = O.bf16_to_f32(a).astype(np.float64).reshape(m, k)
    b64 = O.bf16_to_f32(b).astype(np.float64).reshape(k, n)
    assert normwise_err(c, a64, b64) <= 2.0**-12
    cb = gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=False)
    assert_bf16_out(cb, a64, b64)
    af = O.gen_doubles(m * k, 42).astype(np.float32)
    bf = O.gen_doubles(k * n, 43).astype(np.float32)
    for kernel, tol in (("gemm_tf32", 2.0**-10), ("gemm_f32x3", 2.0**-16)):
        c = gemm(ctx, queues, kernel, af, bf, m, k, n)
        assert normwise_err(c, af.astype(np.float64).reshape(m, k), bf.astype(np.float64).reshape(k, n)) <= tol, kernel


def test_gemm_shapes_bit_identical(ctx, queues, monkeypatch):
    """Every tile shape computes each output with the same per-element MMA chain."""
    m, n, k = 640, 384, 512
    a = O.gen_bf16(m * k, 42)
    b = O.gen_bf16(k * n, 43)
    outs = []
    for shape in "0123":
        monkeypatch.setenv("HCL_GEMM_SHAPE", shape)
        outs.append(gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=True).tobytes())
    assert all(o == outs[0] for o in outs)


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 1024), (300, 200, 136)])
def test_gemm_tf32(ctx, queues, m, n, k):
    a = O.gen_doubles(m * k, 42).astype(np.float32)
    b = O.gen_doubles(k * n, 43).astype(np.float32)
    c = gemm(ctx, queues, "gemm_tf32", a, b, m, k, n)
    assert normwise_err(c, a.astype(np.float64).reshape(m, k), b.astype(np.float64).reshape(k, n)) <= 2.0**-10


# (2560, 2560, 256) takes the 128x128-tile SIMT kernel, the others the 64x64 one
@pytest.mark.parametrize("m,n,k", [(1024, 1024, 1024), (300, 200, 137), (2560, 2560, 256)])
def test_gemm_f32_simt(ctx, queues, m, n, k):
    a = O.gen_doubles(m * k, 42).astype(np.float32)
    b = O.gen_doubles(k * n, 43).astype(np.float32)
    c = gemm(ctx, queues, "gemm_f32", a, b, m, k, n)
    assert normwise_err(c, a.astype(np.float64).reshape(m, k), b.astype(np.float64).reshape(k, n)) <= 2.0**-20


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 1024), (300, 200, 136), (512, 264, 4096)])
def test_gemm_f32x3(ctx, queues, m, n, k):
    a = O.gen_doubles(m * k, 42).astype(np.float32)
    b = O.gen_doubles(k * n, 43).astype(np.float32)
    c = gemm(ctx, queues, "gemm_f32x3", a, b, m, k, n)
    err = normwise_err(c, a.astype(np.float64).reshape(m, k), b.astype(np.float64).reshape(k, n))
    assert err <= 2.0**-16
    if (m, n, k) == (1024, 1024, 1024):  # C1: the default 4-slice K split meets §8(c)'s fp32 bound
        assert err <= 2.0**-20


@pytest.mark.parametrize("kernel", ["gemm_f32", "gemm_f32x3", "gemm_tf32"])
def test_gemm_fp32_partition_invariance(ctx, queues, kernel):
    m, n, k = 1000, 512, 256
    a = O.gen_doubles(m * k, 42).astype(np.float32)
    b = O.gen_doubles(k * n, 43).astype(np.float32)
    whole = gemm(ctx, queues, kernel, a, b, m, k, n)
    for P, w in ((2, None), (4, [1, 2, 3, 4])):
        part = gemm(ctx, queues, kernel, a, b, m, k, n, P=P, weights=w)
        assert whole.tobytes() == part.tobytes(), (kernel, P)


def test_gemm_argument_errors(ctx, queues):
    a = O.gen_bf16(64 * 60, 1)
    with pytest.raises(HaoclError) as e:  # K=60 -> 120-byte rows, not 16-byte aligned
        gemm(ctx, queues, "gemm_bf16", a, O.gen_bf16(60 * 64, 2), 64, 60, 64)
    assert e.value.name == "argument"
    with pytest.raises(HaoclError) as e:  # 3xTF32 needs K % 4 == 0
        gemm(ctx, queues, "gemm_f32x3", np.ones(64 * 62, np.float32), np.ones(62 * 64, np.float32), 64, 62, 64)
    assert e.value.name == "argument"
    with pytest.raises(HaoclError) as e:  # B has the wrong size
        gemm(ctx, queues, "gemm_bf16", O.gen_bf16(64 * 64, 1), O.gen_bf16(64 * 32, 2), 64, 64, 64)
    assert e.value.name == "argument"


def test_gemm_f32_simt_tiles_bit_identical(ctx, queues, monkeypatch):
    m, n, k = 701, 520, 301  # ragged M and K; N % 4 == 0 takes the multistage path
    a = O.gen_doubles(m * k, 42).astype(np.float32)
    b = O.gen_doubles(k * n, 43).astype(np.float32)
    outs = []
    monkeypatch.setenv("HCL_SIMT_KSPLIT", "1")  # one FMA chain per output (the register-prefetch kernel's)
    for ms in "01":  # register-prefetch kernel and the cp.async multistage kernel
        monkeypatch.setenv("HCL_SIMT_MS", ms)
        for t in "012":
            monkeypatch.setenv("HCL_SIMT_TILE", t)
            outs.append(gemm(ctx, queues, "gemm_f32", a, b, m, k, n).tobytes())
    assert all(o == outs[0] for o in outs)
    a64, b64 = a.astype(np.float64).reshape(m, k), b.astype(np.float64).reshape(k, n)
    assert normwise_err(np.frombuffer(outs[0], np.float32).reshape(m, n), a64, b64) <= 2.0**-20


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 1024), (701, 520, 301)])
def test_gemm_f32_simt_ksplit(ctx, queues, monkeypatch, m, n, k):
    """Small grids split K (slices of k-tiles, each an ascending FMA chain, summed
    in slice order): within the fp32 bound, and identical across tile shapes."""
    a = O.gen_doubles(m * k, 46).astype(np.float32)
    b = O.gen_doubles(k * n, 47).astype(np.float32)
    a64, b64 = a.astype(np.float64).reshape(m, k), b.astype(np.float64).reshape(k, n)
    default = gemm(ctx, queues, "gemm_f32", a, b, m, k, n)
    assert normwise_err(default, a64, b64) <= 2.0**-20
    monkeypatch.setenv("HCL_SIMT_KSPLIT", "4")
    outs = []
    for t in "012":
        monkeypatch.setenv("HCL_SIMT_TILE", t)
        outs.append(gemm(ctx, queues, "gemm_f32", a, b, m, k, n).tobytes())
    assert all(o == outs[0] for o in outs)
    assert outs[0] == default.tobytes()  # both sizes take 4 slices by default
    monkeypatch.setenv("HCL_SIMT_KSPLIT", "1")
    one = gemm(ctx, queues, "gemm_f32", a, b, m, k, n)
    assert normwise_err(one, a64, b64) <= 2.0**-20


@pytest.mark.parametrize("kernel,out_f32,tol", [("gemm_bf16", True, 2.0**-12), ("gemm_bf16", False, None),
                                                ("gemm_f32x3", True, 2.0**-16), ("gemm_f32", True, 2.0**-20)])
def test_gemm_full_c2_sampled(ctx, queues, kernel, out_f32, tol):
    """SURVEY.md §8(d) C2 at full size (16384^3, A seed 42, B seed 43): 4096
    seeded (i, j) entries -- a 64 x 64 grid of rows and columns -- against the
    REFERENCE LIBRARY's matmul (fp64, k-ascending, no contraction) of the same
    rounded inputs, with the path's tolerance."""
    s = 16384
    if kernel == "gemm_bf16":
        a, b = O.gen_bf16(s * s, 42), O.gen_bf16(s * s, 43)
        af, bf = O.bf16_to_f32(a).reshape(s, s), O.bf16_to_f32(b).reshape(s, s)
    else:
        a, b = O.gen_doubles(s * s, 42).astype(np.float32), O.gen_doubles(s * s, 43).astype(np.float32)
        af, bf = a.reshape(s, s), b.reshape(s, s)
    c = gemm(ctx, queues, kernel, a, b, s, s, s, out_f32=out_f32)
    rng = np.random.default_rng(11)
    ii, jj = np.sort(rng.choice(s, 64, replace=False)), np.sort(rng.choice(s, 64, replace=False))
    a64, b64 = af[ii].astype(np.float64), np.ascontiguousarray(bf[:, jj].astype(np.float64))
    rc, work, out = O.ref_execute("matmul", [("in", a64), ("in", b64), ("out", None), ("s", 64), ("s", s), ("s", 64)],
                                  {2: 64 * 64 * 8}, threads=os.cpu_count() or 1)
    assert rc == 0 and work == 2 * 64 * s * 64
    c64 = out[2].view(np.float64).reshape(64, 64)
    assert np.abs(c64 - a64 @ b64).max() <= 2.0**-40 * (np.abs(a64) @ np.abs(b64)).max()  # the oracle agrees
    got = c[np.ix_(ii, jj)].astype(np.float64)
    scale = np.abs(a64) @ np.abs(b64)
    if tol is not None:
        assert float((np.abs(got - c64) / scale).max()) <= tol
    else:  # bf16 output: the 2^-10 product bound plus one bf16 rounding
        assert (np.abs(got - c64) <= 2.0**-10 * (1 + 2.0**-8) * scale + 2.0**-8 * np.abs(c64)).all()


def test_gemm_f32x3_ksplit(ctx, queues, monkeypatch):
    """Optional K split (HCL_GEMM_KSPLIT): slices summed in order -- within the
    3xTF32 tolerance and bit-identical across row partitions."""
    monkeypatch.setenv("HCL_GEMM_KSPLIT", "4")
    m, n, k = 1024, 512, 1024
    a = O.gen_doubles(m * k, 42).astype(np.float32)
    b = O.gen_doubles(k * n, 43).astype(np.float32)
    whole = gemm(ctx, queues, "gemm_f32x3", a, b, m, k, n)
    assert normwise_err(whole, a.astype(np.float64).reshape(m, k), b.astype(np.float64).reshape(k, n)) <= 2.0**-16
    part = gemm(ctx, queues, "gemm_f32x3", a, b, m, k, n, P=4, weights=[1, 2, 3, 4])
    assert whole.tobytes() == part.tobytes()


@pytest.mark.parametrize("m,k,n,ks", [(1024, 1024, 1024, ""), (300, 96, 260, "3"), (257, 2048, 132, "1"),
                                       (130, 100, 68, "")])
def test_gemm_f32x3_segments_bit_identical(ctx, queues, monkeypatch, m, k, n, ks):
    """K a multiple of 32: the split stores [hi | lo] once per operand and the
    GEMM's producer reads A' = [hi|hi|lo], B' = [hi|lo|hi] segment by segment
    (HCL_GEMM_SEG, default) -- the same MMAs in the same order as the
    materialised 3K layout, so C is bit-identical (K = 100: no segments)."""
    if ks:
        monkeypatch.setenv("HCL_GEMM_KSPLIT", ks)
    a = O.gen_doubles(m * k, 44).astype(np.float32)
    b = O.gen_doubles(k * n, 45).astype(np.float32)
    monkeypatch.setenv("HCL_GEMM_SEG", "0")
    want = gemm(ctx, queues, "gemm_f32x3", a, b, m, k, n)
    monkeypatch.setenv("HCL_GEMM_SEG", "1")
    got = gemm(ctx, queues, "gemm_f32x3", a, b, m, k, n)
    assert got.tobytes() == want.tobytes()
    assert normwise_err(got, a.astype(np.float64).reshape(m, k), b.astype(np.float64).reshape(k, n)) <= 2.0**-16


@pytest.mark.parametrize("one", ["1", "0"])
def test_gemm_bf16_b_multicast_bit_identical(ctx, queues, monkeypatch, one):
    """HCL_GEMM_MC=1: clusters of two CTA pairs on vertically adjacent tiles, each
    B atom loaded once and multicast to both pairs (TMA .multicast::cluster) --
    the same MMAs in the same order, so C is bit-identical to the default path."""
    m = n = 4096
    k = 1024
    a = O.gen_bf16(m * k, 42)
    b = O.gen_bf16(k * n, 43)
    monkeypatch.setenv("HCL_GEMM_ONE", one)
    monkeypatch.setenv("HCL_GEMM_MC", "0")
    want = gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=False)  # C2's bf16-out (TMA-store) path
    monkeypatch.setenv("HCL_GEMM_MC", "1")
    got = gemm(ctx, queues, "gemm_bf16", a, b, m, k, n, out_f32=False)
    assert got.tobytes() == want.tobytes()
