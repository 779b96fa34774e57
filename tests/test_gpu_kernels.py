"""Kernel-level parity on the GPU (``-m gpu``): the production tcgen05 GEMM,
the per-row quantizer and the attention kernel, called through the C ABI and
compared element by element with the CPU oracle / brute force."""
import numpy as np
import pytest

import oracle
from paper_2010_13382_b200 import fastformers as ffb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _pitched(arr_np, dtype, align_elems):
    """Copy a [R, K] numpy array into a CUDA tensor whose row pitch is K rounded
    up to align_elems (16-byte rows), returning the [R, K] view."""
    R, K = arr_np.shape
    ld = (K + align_elems - 1) // align_elems * align_elems
    t = torch.zeros((R, ld), dtype=dtype, device="cuda")
    t[:, :K] = torch.from_numpy(arr_np).to("cuda")
    return t[:, :K]


# every GEMM shape of BASELINE configs[0..4] (SURVEY 8(a) shape table) plus ragged M / N / K
I8_SHAPES = [
    (128, 128, 128), (128, 384, 128), (128, 192, 128), (128, 128, 64), (128, 256, 128), (128, 128, 256),  # C1
    (200, 936, 312), (333, 312, 312), (130, 1200, 312), (129, 312, 1200),                                 # C2
    (300, 702, 312), (260, 624, 312), (257, 312, 234), (140, 900, 312), (140, 312, 900),                   # C2 pruned
    (1000, 1536, 768), (520, 768, 512), (384, 768, 1536),                                                   # C3
    (256, 2304, 768), (256, 768, 3072), (300, 1024, 4096), (300, 4096, 1024),                              # C4/C5
    (1, 16, 16), (17, 8, 32), (4096, 1536, 768),
]


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("M,N,K", I8_SHAPES)
def test_gemm_i8_int32_accumulators_bit_exact(M, N, K, pair):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.integers(-127, 128, (M, K), dtype=np.int8)
    W = rng.integers(-127, 128, (N, K), dtype=np.int8)
    C = ffb.gemm(_pitched(A, torch.int8, 16), _pitched(W, torch.int8, 16), out_mode=0, cta_pair=pair)
    torch.cuda.synchronize()
    got = C.cpu().numpy()
    if M * N * K <= 3e8:
        ref = oracle.gemm_s8(A, W)
    else:  # brute force too slow on CPU at this size: cuBLASLt int8 as the independent reference
        ref = torch._int_mm(torch.from_numpy(A).cuda(), torch.from_numpy(W).cuda().t().contiguous()).cpu().numpy() \
            if M > 16 and K % 8 == 0 and N % 8 == 0 else (A.astype(np.int64) @ W.astype(np.int64).T).astype(np.int32)
    assert np.array_equal(got, ref), f"max diff {np.abs(got.astype(np.int64) - ref).max()}"


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (200, 936, 312), (1000, 1536, 768), (300, 768, 3072),
                                   (129, 1200, 312), (77, 1024, 4096)])
def test_gemm_f16_fp32_accumulators_within_bound(M, N, K, pair):
    rng = np.random.default_rng(K)
    A = np.float16(rng.standard_normal((M, K)))
    W = np.float16(rng.standard_normal((N, K)) * 0.05)
    C = ffb.gemm(_pitched(A, torch.float16, 8), _pitched(W, torch.float16, 8), out_mode=0, cta_pair=pair)
    torch.cuda.synchronize()
    got = C.cpu().numpy().astype(np.float64)
    A64, W64 = A.astype(np.float64), W.astype(np.float64)
    ref = A64 @ W64.T
    bound = K * 2.0 ** -24 * (np.abs(A64) @ np.abs(W64).T) + 1e-30
    assert np.all(np.abs(got - ref) <= bound), np.max(np.abs(got - ref) / bound)


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("act", [-1, 0, 1, 2])
def test_gemm_epilogues(act, pair):
    rng = np.random.default_rng(5 + act)
    M, N, K = 300, 640, 512
    A = rng.integers(-127, 128, (M, K), dtype=np.int8)
    W = rng.integers(-127, 128, (N, K), dtype=np.int8)
    sx = (rng.random(M) * 0.01 + 1e-3).astype(np.float32)
    sw = (rng.random(N) * 0.001 + 1e-4).astype(np.float32)
    b = (rng.standard_normal(N) * 0.1).astype(np.float32)
    out = ffb.gemm(_pitched(A, torch.int8, 16), _pitched(W, torch.int8, 16), out_mode=1,
                   bias=torch.from_numpy(b).cuda(), sx=torch.from_numpy(sx).cuda(), sw=torch.from_numpy(sw).cuda(),
                   act=act, cta_pair=pair)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    acc = A.astype(np.int64) @ W.astype(np.int64).T
    y = acc * (sx[:, None].astype(np.float64) * sw[None, :]) + b[None, :]
    yact = oracle.act(y.astype(np.float32), act).reshape(y.shape) if act >= 0 else y
    ref = np.float16(yact).astype(np.float64)
    # one fp16 ulp of slack (fp32 epilogue vs fp64 reference before the final R16)
    assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -10 + 2.0 ** -24 * 4), np.abs(got - ref).max()


def test_quant_rows_bit_exact_vs_oracle():
    rng = np.random.default_rng(11)
    for M, K in [(64, 312), (33, 1536), (5, 4096), (7, 234)]:
        x = np.float16(rng.standard_normal((M, K)) * rng.uniform(0.01, 10, (M, 1)))
        x[0] = 0
        x[1, :4] = np.float16([127.0, 62.5, 63.5, -62.5])
        x[1, 4:] = 0
        # ties of x/s with s = 3 (x * rcp(s) lands one ulp off the tie)
        x[2, :6] = np.float16([381.0, 10.5, 4.5, 13.5, -10.5, 7.5])
        x[2, 6:] = np.float16(rng.integers(-254, 254, K - 6) * 1.5)
        q, s = ffb.quant_rows(_pitched(x, torch.float16, 8))
        torch.cuda.synchronize()
        rq, rs = oracle.q8row(x.astype(np.float32))
        assert np.array_equal(s.cpu().numpy(), rs)
        assert np.array_equal(q.cpu().numpy(), rq)


@pytest.mark.parametrize("B,S,A,d,ragged", [(2, 40, 3, 64, True), (2, 128, 12, 26, True), (1, 300, 2, 64, True),
                                             (2, 512, 2, 64, True), (3, 128, 8, 64, False), (1, 7, 1, 64, False),
                                             (1, 256, 4, 32, True)])
def test_attention_matches_oracle(B, S, A, d, ragged):
    rng = np.random.default_rng(S + A + d)
    qkv = np.float16(rng.standard_normal((B * S, 3 * A * d)) * 1.5)
    mask = np.ones((B, S), np.int32)
    if ragged:
        for b in range(B):
            mask[b, rng.integers(max(1, S // 4), S + 1):] = 0
        if S > 8:
            mask[0, S // 2] = 0  # a hole, not only a padded tail
    ctx = ffb.attention(torch.from_numpy(qkv).cuda(), torch.from_numpy(mask).cuda(), A, d, impl=1)
    torch.cuda.synchronize()
    got = ctx.cpu().numpy().astype(np.float64)
    ref = oracle.attention(qkv.astype(np.float32), mask, A, d).astype(np.float64)
    ref64 = oracle.attention(qkv.astype(np.float32), mask, A, d, mode=oracle.MODE_REF64).astype(np.float64)
    err = np.abs(got - ref)
    # fp16 output: one rounding of ctx plus rare one-ulp flips of P16
    assert err.max() <= 4e-3 + 4e-3 * np.abs(ref).max(), err.max()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-3
    assert np.abs(got - ref64).max() <= 2e-2


@pytest.mark.parametrize("B,S,A,ragged,d", [(2, 128, 8, False, 64), (3, 128, 4, True, 64), (2, 40, 3, True, 64),
                                            (1, 7, 2, False, 64), (4, 32, 2, True, 64), (1, 1, 1, False, 64),
                                            (2, 64, 12, True, 64), (3, 128, 16, False, 64),
                                            # head_dim <= 32 padded to 32 (TMA-aligned head slices)
                                            (2, 128, 8, False, 32), (1, 1, 1, False, 32), (3, 128, 12, True, 32),
                                            (2, 64, 4, True, 16), (2, 40, 6, True, 24)])
def test_attention_tcgen05_matches_oracle(B, S, A, ragged, d):
    """The tcgen05/TMEM attention kernel (head_dim 64 or even <= 32, S <= 128)."""
    rng = np.random.default_rng(100 + S + A + d)
    qkv = np.float16(rng.standard_normal((B * S, 3 * A * d)) * 1.5)
    mask = np.ones((B, S), np.int32)
    if ragged:
        for b in range(B):
            mask[b, rng.integers(max(1, S // 4), S + 1):] = 0
        mask[0, S // 2] = 0
    mask[:, 0] = 1
    ctx = ffb.attention(torch.from_numpy(qkv).cuda(), torch.from_numpy(mask).cuda(), A, d, impl=2)
    torch.cuda.synchronize()
    got = ctx.cpu().numpy().astype(np.float64)
    ref = oracle.attention(qkv.astype(np.float32), mask, A, d).astype(np.float64)
    err = np.abs(got - ref)
    assert err.max() <= 4e-3 + 4e-3 * np.abs(ref).max(), err.max()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-3
    # and the same as the mma.sync kernel up to rounding
    ctx1 = ffb.attention(torch.from_numpy(qkv).cuda(), torch.from_numpy(mask).cuda(), A, d, impl=1).cpu().numpy()
    assert np.abs(ctx1.astype(np.float64) - got).max() <= 4e-3 + 4e-3 * np.abs(ref).max()


@pytest.mark.parametrize("B,S,A,ragged", [(2, 256, 4, True), (1, 512, 3, True), (2, 512, 2, False), (3, 129, 2, True),
                                          (2, 300, 3, True), (1, 384, 2, False), (4, 200, 12, True), (1, 511, 1, True)])
def test_attention_long_tcgen05_matches_oracle(B, S, A, ragged):
    """The tcgen05 attention for 128 < S <= 512 (attention_long.cu: max over
    all key chunks, then e = exp(s - max) and l, then P16 = R16(e / l) chunk
    by chunk -- the oracle's order, DESIGN R9), head_dim 64, ragged masks
    with holes, partial last chunks and query blocks."""
    d = 64
    rng = np.random.default_rng(700 + S + A + B)
    qkv = np.float16(rng.standard_normal((B * S, 3 * A * d)) * 1.5)
    mask = np.ones((B, S), np.int32)
    if ragged:
        for b in range(B):
            mask[b, rng.integers(max(1, S // 4), S + 1):] = 0
        mask[0, S // 2] = 0
    mask[:, 0] = 1
    ctx = ffb.attention(torch.from_numpy(qkv).cuda(), torch.from_numpy(mask).cuda(), A, d, impl=2)
    torch.cuda.synchronize()
    got = ctx.cpu().numpy().astype(np.float64)
    ref = oracle.attention(qkv.astype(np.float32), mask, A, d).astype(np.float64)
    err = np.abs(got - ref)
    assert err.max() <= 4e-3 + 4e-3 * np.abs(ref).max(), err.max()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-3
    # and the same as the mma.sync kernel (online max / sum) up to rounding
    ctx1 = ffb.attention(torch.from_numpy(qkv).cuda(), torch.from_numpy(mask).cuda(), A, d, impl=1).cpu().numpy()
    assert np.abs(ctx1.astype(np.float64) - got).max() <= 4e-3 + 4e-3 * np.abs(ref).max()


@pytest.mark.parametrize("B,S,A,ragged,d", [(2, 128, 8, False, 64), (3, 128, 4, True, 64), (2, 40, 3, True, 64),
                                            (1, 7, 2, False, 64), (1, 1, 1, False, 64), (5, 128, 8, True, 64),
                                            (150, 16, 2, True, 64), (2, 128, 8, True, 32), (3, 128, 16, False, 32),
                                            (1, 1, 8, False, 32)])
def test_attention_fused_requant(B, S, A, ragged, d):
    """a3 + a4 fused (the int8-layer path): ctx within the attention bound of
    the oracle, and the s8 rows / scales bit-exact Q8row of the kernel's own
    fp16 ctx (DESIGN R6-R8, R12); head_dim 64 (<= 8 heads per sequence) and
    32 (<= 16 heads)."""
    rng = np.random.default_rng(300 + S + A + B + d)
    qkv = np.float16(rng.standard_normal((B * S, 3 * A * d)) * 1.5)
    mask = np.ones((B, S), np.int32)
    if ragged:
        for b in range(B):
            mask[b, rng.integers(max(1, S // 4), S + 1):] = 0
        mask[0, S // 2] = 0
    mask[:, 0] = 1
    qkv_d, mask_d = torch.from_numpy(qkv).cuda(), torch.from_numpy(mask).cuda()
    ctx, q, sc = ffb.attention_q8(qkv_d, mask_d, A, d)
    torch.cuda.synchronize()
    got = ctx.cpu().numpy()
    ref = oracle.attention(qkv.astype(np.float32), mask, A, d).astype(np.float64)
    assert np.abs(got.astype(np.float64) - ref).max() <= 4e-3 + 4e-3 * np.abs(ref).max()
    rq, rs = oracle.q8row(got.astype(np.float32))
    np.testing.assert_array_equal(q.cpu().numpy(), rq)
    np.testing.assert_array_equal(sc.cpu().numpy(), rs)
    # without the fp16 copy: the same s8 rows
    _, q2, s2 = ffb.attention_q8(qkv_d, mask_d, A, d, with_ctx16=False)
    assert torch.equal(q2, q) and torch.equal(s2, sc)
