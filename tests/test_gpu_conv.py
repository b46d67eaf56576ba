"""3x3 conv (config C5) parity against the fp64 oracle of the same bf16
inputs (exact products, c -> r -> s order; oracle ho_conv3x3_point and a numpy
fp64 full reference). Tolerance (normwise, |out - ref| / sum|x||w|):
2^-12 for fp32 output, 2^-8 for bf16 output. Outputs are bit-identical for
every batch partition (P in {1, 2, 4}, even and uneven weights)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def queues(ctx):
    qs = [ctx.create_queue(g) for g in ctx.get_device_ids()[:4]]
    yield qs
    for q in qs:
        ctx.release(q)


def ref_conv(x, w):
    n, h, wd, c = x.shape
    k = w.shape[0]
    xp = np.zeros((n, h + 2, wd + 2, c))
    xp[:, 1:-1, 1:-1] = x
    out = np.zeros((n, h, wd, k))
    scale = np.zeros((n, h, wd, k))
    for r in range(3):
        for s in range(3):
            patch = xp[:, r:r + h, s:s + wd, :]
            out += patch @ w[:, r, s, :].T
            scale += np.abs(patch) @ np.abs(w[:, r, s, :]).T
    return out, scale


def run(ctx, queues, n, h, wd, c, k, out_f32, P=1, weights=None, padded=None):
    from paper_2005_08466_b200.conv import Conv3x3

    xb = O.gen_bf16(n * h * wd * c, 42).reshape(n, h, wd, c)
    wb = O.gen_bf16(k * 9 * c, 43).reshape(k, 3, 3, c)
    cv = Conv3x3(ctx, queues[:P], n, h, wd, c, k, out_f32=out_f32, padded=padded)
    cv.load(xb, wb, weights)
    cv.run()
    got = cv.output().copy()
    cv.close()
    return xb, wb, got


@pytest.mark.parametrize("n,h,wd,c,out_f32", [(2, 16, 16, 64, True), (3, 7, 37, 128, True), (2, 12, 30, 64, False),
                                             (3, 9, 50, 64, False), (2, 5, 224, 64, False), (1, 33, 17, 64, True),
                                             (2, 17, 9, 64, False)])
def test_conv_matches_fp64_reference(ctx, queues, n, h, wd, c, out_f32):
    k = 128
    xb, wb, got = run(ctx, queues, n, h, wd, c, k, out_f32)
    x = O.bf16_to_f32(xb).astype(np.float64)
    w = O.bf16_to_f32(wb).astype(np.float64)
    ref, scale = ref_conv(x, w)
    err = (np.abs(got - ref) / np.maximum(scale, 1e-30)).max()
    assert err <= (2.0**-12 if out_f32 else 2.0**-8)
    # spot-check against the C oracle (fixed c -> r -> s order)
    rng = np.random.default_rng(0)
    for _ in range(20):
        i, y, xx, ko = (int(rng.integers(0, v)) for v in (n, h, wd, k))
        o = O.conv3x3_point(xb.reshape(-1), wb.reshape(-1), h, wd, c, k, i, y, xx, ko)
        assert abs(got[i, y, xx, ko] - o) <= (2.0**-12 if out_f32 else 2.0**-8) * max(scale[i, y, xx, ko], 1e-30)


@pytest.mark.parametrize("n,h,wd,out_f32", [(2, 16, 16, True), (2, 12, 30, False), (3, 33, 47, False),
                                           (1, 224, 224, False)])
def test_conv_nhwc_equals_padded_path(ctx, queues, n, h, wd, out_f32):
    """conv3x3_nhwc (halo tiles straight from NHWC, TMA zero fill) and the
    padded kernel (conv_pad_nhwc + conv3x3) issue the same per-output MMA chain
    (taps r, s, then 16-channel steps): outputs bit-identical, ragged tiles too."""
    _, _, a = run(ctx, queues, n, h, wd, 64, 128, out_f32, padded=False)
    _, _, b = run(ctx, queues, n, h, wd, 64, 128, out_f32, padded=True)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("P,weights", [(2, None), (4, None), (4, [1, 3, 2, 2])])
def test_conv_partition_invariance(ctx, queues, P, weights):
    n, h, wd, c, k = 8, 10, 20, 64, 128
    _, _, whole = run(ctx, queues, n, h, wd, c, k, True)
    _, _, part = run(ctx, queues, n, h, wd, c, k, True, P=P, weights=weights)
    assert whole.tobytes() == part.tobytes()


def test_conv_full_c5_sampled(ctx, queues):
    """SURVEY.md §8(d) C5 at full size (batch 256, 224 x 224, 64 -> 128, bf16
    output): 4096 seeded output points -- a quarter of them on the padded
    border -- against the C oracle's fp64 direct conv of the same bf16 inputs."""
    from paper_2005_08466_b200.conv import Conv3x3

    n, h, wd, c, k = 256, 224, 224, 64, 128
    xb = O.gen_bf16(n * h * wd * c, 42)
    wb = O.gen_bf16(k * 9 * c, 43)
    cv = Conv3x3(ctx, queues[:1], n, h, wd, c, k, out_f32=False)
    try:
        cv.load(xb.reshape(n, h, wd, c), wb.reshape(k, 3, 3, c))
        cv.run()
        cv.finish()
        raw = ctx.enqueue_read_buffer(queues[0], cv.b_out).view(np.uint16)
    finally:
        cv.close()
    rng = np.random.default_rng(5)
    m = 4096
    ni, yi, xi, ki = (rng.integers(0, v, m) for v in (n, h, wd, k))
    edge = rng.integers(0, 4, m)  # first quarter: pin y or x to a border
    yi[: m // 8] = np.where(edge[: m // 8] & 1, h - 1, 0)
    xi[m // 8: m // 4] = np.where(edge[m // 8: m // 4] & 1, wd - 1, 0)
    x = xb.reshape(n, h, wd, c)  # bf16 bits; converted per patch
    w = np.abs(O.bf16_to_f32(wb).reshape(k, 3, 3, c).astype(np.float64))
    for i, y, xx, ko in zip(ni, yi, xi, ki):
        i, y, xx, ko = int(i), int(y), int(xx), int(ko)
        got = float(O.bf16_to_f32(raw[((i * h + y) * wd + xx) * k + ko: ((i * h + y) * wd + xx) * k + ko + 1])[0])
        want = O.conv3x3_point(xb, wb, h, wd, c, k, i, y, xx, ko)
        scale = 0.0
        for r in range(3):
            for s in range(3):
                yy, xs = y + r - 1, xx + s - 1
                if 0 <= yy < h and 0 <= xs < wd:
                    scale += float(np.abs(O.bf16_to_f32(x[i, yy, xs]).astype(np.float64)) @ w[ko, r, s])
        assert abs(got - want) <= 2.0**-8 * max(scale, 1e-30), (i, y, xx, ko, got, want)
