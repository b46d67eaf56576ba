"""In-process partitioned launches over REAL distinct GPUs (NVLink peer copies
between devices): skipped on a single-GPU box, run by the multi-GPU check
(`gpurun --gpus 2|4`). The same parity bars as the logical-device tests:
bit-identical to the whole launch / the reference digests."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mctx(ctx):
    """The session context; its devices 3.. are GPU 0 and one per other GPU."""
    ords = ctx.cuda_ordinals
    if len(set(ords)) < 2:
        pytest.skip("needs >= 2 GPUs")
    ids = ctx.get_device_ids()
    ctx.multi_ids = [ids[3]] + ids[4:]
    return ctx


def test_matmul_digest_over_gpus(mctx, golden):
    qs = [mctx.create_queue(g) for g in mctx.multi_ids]
    n = 512
    a, b = O.gen_doubles(n * n, 42), O.gen_doubles(n * n, 43)
    prog = mctx.create_program("core")
    k = mctx.create_kernel(prog, "matmul")
    ba, bb, bc = mctx.create_buffer(a.nbytes), mctx.create_buffer(b.nbytes), mctx.create_buffer(n * n * 8)
    mctx.enqueue_write_buffer(qs[0], ba, a)
    mctx.enqueue_write_buffer(qs[0], bb, b)
    for i, v in enumerate([ba, bb, bc, n, n, n]):
        mctx.set_kernel_arg(k, i, v)
    mctx.enqueue_ndrange_partitioned(k, (n, n, 1), 2, qs)
    for q in qs:
        mctx.finish(q)
    out = mctx.enqueue_read_buffer(qs[-1], bc)
    assert f"{O.fnv1a(out):016x}" == golden["digests"]["matmul_512"]


def test_gemm_and_knn_refsplit_over_gpus(mctx, golden):
    qs = [mctx.create_queue(g) for g in mctx.multi_ids]
    m, n, kk = 2048, 1024, 512
    a, b = O.gen_bf16(m * kk, 1), O.gen_bf16(kk * n, 2)
    prog = mctx.create_program("b200")
    k = mctx.create_kernel(prog, "gemm_bf16")
    ba, bb, bc = mctx.create_buffer(a.nbytes), mctx.create_buffer(b.nbytes), mctx.create_buffer(m * n * 4)
    mctx.enqueue_write_buffer(qs[0], ba, a)
    mctx.enqueue_write_buffer(qs[0], bb, b)
    for i, v in enumerate([ba, bb, bc, m, kk, n, 1]):
        mctx.set_kernel_arg(k, i, v)
    mctx.enqueue_ndrange_kernel(qs[0], k, (m, n, 1), 2)
    mctx.finish(qs[0])
    whole = mctx.enqueue_read_buffer(qs[0], bc).tobytes()
    mctx.enqueue_ndrange_partitioned(k, (m, n, 1), 2, qs, [3, 1] + [2] * (len(qs) - 2))
    for q in qs:
        mctx.finish(q)
    assert mctx.enqueue_read_buffer(qs[1], bc).tobytes() == whole

    R, Q, D, K = 10**5, 10**3, 16, 10
    rf, qq = O.gen_doubles(R * D, 42), O.gen_doubles(Q * D, 43)
    kn = mctx.create_kernel(prog, "knn_refsplit")
    br, bq = mctx.create_buffer(rf.nbytes), mctx.create_buffer(qq.nbytes)
    bi, bd = mctx.create_buffer(Q * K * 4), mctx.create_buffer(Q * K * 8)
    mctx.enqueue_write_buffer(qs[0], br, rf)
    mctx.enqueue_write_buffer(qs[0], bq, qq)
    for i, v in enumerate([br, bq, R, Q, D, K, bi, bd]):
        mctx.set_kernel_arg(kn, i, v)
    mctx.enqueue_ndrange_partitioned(kn, (R, 1, 1), 1, qs)
    for q in qs:
        mctx.finish(q)
    idx = mctx.enqueue_read_buffer(qs[0], bi)
    dist = mctx.enqueue_read_buffer(qs[0], bd)
    assert f"{O.fnv1a(dist, O.fnv1a(idx)):016x}" == golden["digests"][f"knn_{R}x{Q}x{D}k{K}"]
