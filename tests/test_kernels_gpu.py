"""Kernel numerics on the B200: every libhx kernel against a plain PyTorch fp32
reference of the same op on the same bf16 inputs (tolerances stated inline)."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU hosts, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2507_00394_b200.runtime import kernels as K  # noqa: E402

DEV = "cuda"


def rel_err(got, want):
    got, want = got.float(), want.float()
    return ((got - want).abs().max() / want.abs().max().clamp_min(1e-30)).item()


def rnd(*shape, scale=1.0, seed=0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return (torch.randn(*shape, generator=g, device=DEV) * scale).to(torch.bfloat16)


GEMM_SHAPES = [(256, 256, 256), (1024, 768, 256), (304, 200, 72), (128, 2048, 512), (2048, 1024, 1024),
               # enough 256x256 M-block pairs for the 2-CTA multicast path (incl. ragged edges)
               (4096, 2560, 512), (4000, 2504, 200)]


@pytest.mark.parametrize("M,N,Kd", GEMM_SHAPES)
def test_gemm_forward_layout(M, N, Kd):
    # y = x @ w : A K-major, B N-major; bf16 out.  tol: 1e-2 of max|ref| (bf16 rounding)
    x, w = rnd(M, Kd, seed=1), rnd(Kd, N, scale=Kd ** -0.5, seed=2)
    y = K.linear(x, w)
    torch.cuda.synchronize()
    assert rel_err(y, x.float() @ w.float()) < 1e-2


@pytest.mark.parametrize("M,N,Kd", GEMM_SHAPES)
def test_gemm_dx_layout(M, N, Kd):
    # dx = dy @ w^T : A K-major, B K-major
    dy, w = rnd(M, Kd, seed=3), rnd(N, Kd, scale=Kd ** -0.5, seed=4)
    dx = K.linear_dx(dy, w)
    torch.cuda.synchronize()
    assert rel_err(dx, dy.float() @ w.float().t()) < 1e-2


@pytest.mark.parametrize("M,N,Kd", GEMM_SHAPES)
def test_gemm_dw_layout_accumulates(M, N, Kd):
    # acc += x^T dy : A M-major, B N-major, f32 accumulate.  tol 1e-4 (fp32 accum of bf16 inputs)
    x, dy = rnd(Kd, M, seed=5), rnd(Kd, N, seed=6)
    acc = torch.randn(M, N, device=DEV)
    want = acc + x.float().t() @ dy.float()
    K.linear_dw(x, dy, acc, accumulate=True)
    torch.cuda.synchronize()
    assert rel_err(acc, want) < 1e-4


@pytest.mark.parametrize("M,N,Kd", [(2048, 8192, 8192), (4096, 4000, 12008)])
def test_gemm_dw_split_k(M, N, Kd):
    # long-K weight gradients with 256 tiles on 74 pairs take the 2-slice pair
    # kernel (slices added into acc with red.global.add); ragged N and K
    x, dy = rnd(Kd, M, seed=15), rnd(Kd, N, seed=16)
    acc = torch.randn(M, N, device=DEV)
    want = acc + x.float().t() @ dy.float()
    K.linear_dw(x, dy, acc, accumulate=True)
    torch.cuda.synchronize()
    assert rel_err(acc, want) < 1e-4


@pytest.mark.parametrize("M,N,Kd", [(256, 1024, 100), (512, 2048, 36), (4096, 4096, 1000), (128, 64, 1)])
def test_gemm_dw_ragged_k(M, N, Kd):
    # weight gradient over a ragged MLP row slab (K not a multiple of 8): the
    # K tail is read through TMA out-of-bounds zero fill
    x, dy = rnd(Kd, M, seed=17), rnd(Kd, N, seed=18)
    acc = torch.randn(M, N, device=DEV)
    want = acc + x.float().t() @ dy.float()
    K.linear_dw(x, dy, acc, accumulate=True)
    torch.cuda.synchronize()
    assert rel_err(acc, want) < 1e-4


def test_attention_delta_matches_rowsum():
    # D = rowsum(dO * O) per (batch, head, query), fp32
    s, b, heads, d = 300, 2, 3, 64
    o, do = rnd(s * b, heads * d, seed=19), rnd(s * b, heads * d, seed=20)
    delta = torch.empty(b * heads * s, device=DEV)
    K.attention_delta(o, do, s, b, heads, delta)
    torch.cuda.synchronize()
    want = (o.float() * do.float()).view(s, b, heads, d).sum(-1).permute(1, 2, 0).reshape(-1)
    assert rel_err(delta, want) < 1e-5


@pytest.mark.parametrize("T,Kd,N", [(4096, 512, 1024), (4000, 256, 1000), (8192, 1024, 2056)])
def test_gemm_pair_kernel_epilogues(T, Kd, N):
    # shapes with >= 32 tile pairs take the cta_group::2 kernel, whose bf16 epilogues
    # (store, +residual, GeLU with its pre-activation, x GeLU') leave through smem and
    # TMA stores; ragged M and N exercise the clipped boxes.  tol 1e-2 of max|ref|
    x, w = rnd(T, Kd, seed=21), rnd(Kd, N, scale=Kd ** -0.5, seed=22)
    ref = x.float() @ w.float()
    y = K.linear(x, w)
    m1 = torch.empty(T, N, dtype=torch.bfloat16, device=DEV)
    g = torch.empty_like(m1)
    K.linear_gelu(x, w, m1, g)
    resid = rnd(T, N, seed=23)
    yr = K.linear_resid(x, w, resid)
    w2 = rnd(Kd, N, scale=N ** -0.5, seed=24)
    dy = rnd(T, N, seed=25)
    m1b = rnd(T, Kd, seed=26)
    dm = torch.empty(T, Kd, dtype=torch.bfloat16, device=DEV)
    K.linear_dx_dgelu(dy, w2, m1b, dm)
    torch.cuda.synchronize()
    assert rel_err(y, ref) < 1e-2
    assert rel_err(m1, ref) < 1e-2
    assert rel_err(g, torch.nn.functional.gelu(ref)) < 1e-2
    assert rel_err(yr, ref + resid.float()) < 1e-2
    mf = m1b.float()
    gelu_grad = 0.5 * (1 + torch.erf(mf / math.sqrt(2))) + mf * torch.exp(-0.5 * mf * mf) / math.sqrt(2 * math.pi)
    assert rel_err(dm, (dy.float() @ w2.float().t()) * gelu_grad) < 1e-2


@pytest.mark.parametrize("T,N", [(8192, 1024), (512, 256)])
def test_gelu_epilogues_to_the_bf16_ulp(T, N):
    # identity weights make every accumulator exactly the bf16 input, so the fused
    # GeLU / GeLU' epilogue math (A&S erf, bare MUFU ex2 / rcp) is checked element by
    # element: within one bf16 ulp of the exact erf GeLU of the same value.
    # (8192, 1024) takes the cta_group::2 kernel, (512, 256) the single-CTA one.
    g_ = torch.Generator(device=DEV).manual_seed(31)
    x = (torch.rand(T, N, generator=g_, device=DEV) * 14 - 7).to(torch.bfloat16)   # [-7, 7)
    x[0, :8] = torch.tensor([0.0, -0.0, 1e-3, -1e-3, 40.0, -40.0, 1e-30, -6.5])
    eye = torch.eye(N, device=DEV, dtype=torch.bfloat16)
    m1 = torch.empty(T, N, dtype=torch.bfloat16, device=DEV)
    g = torch.empty_like(m1)
    K.linear_gelu(x, eye, m1, g)
    dy = rnd(T, N, seed=32)
    dm = torch.empty(T, N, dtype=torch.bfloat16, device=DEV)
    K.linear_dx_dgelu(dy, eye, x, dm)
    torch.cuda.synchronize()
    xf = x.float().double()
    assert torch.equal(m1, x)
    want_g = torch.nn.functional.gelu(xf)
    ulp = lambda v: v.abs().clamp_min(1e-30) * 2.0 ** -8  # noqa: E731
    assert ((g.double() - want_g).abs() <= ulp(want_g) + 1e-6).all()
    grad = 0.5 * (1 + torch.erf(xf / math.sqrt(2))) + xf * torch.exp(-0.5 * xf * xf) / math.sqrt(2 * math.pi)
    want_dm = dy.double() * grad
    assert ((dm.double() - want_dm).abs() <= ulp(want_dm) + 1e-6).all()


def test_gemm_epilogues():
    T, Kd, N = 512, 256, 1024
    x, w = rnd(T, Kd, seed=7), rnd(Kd, N, scale=Kd ** -0.5, seed=8)
    ref = x.float() @ w.float()
    m1 = torch.empty(T, N, dtype=torch.bfloat16, device=DEV)
    g = torch.empty_like(m1)
    K.linear_gelu(x, w, m1, g)
    resid = rnd(T, N, seed=9)
    yr = K.linear_resid(x, w, resid)
    w2 = rnd(Kd, N, scale=N ** -0.5, seed=10)  # used as [i=Kd, o=N]: dx = dy[T,N] @ w2^T
    dy = rnd(T, N, seed=11)
    dm = torch.empty(T, Kd, dtype=torch.bfloat16, device=DEV)
    m1b = rnd(T, Kd, seed=12)
    K.linear_dx_dgelu(dy, w2, m1b, dm)
    torch.cuda.synchronize()
    assert rel_err(m1, ref) < 1e-2
    assert rel_err(g, torch.nn.functional.gelu(ref)) < 1e-2
    assert rel_err(yr, ref + resid.float()) < 1e-2
    mf = m1b.float()
    gelu_grad = 0.5 * (1 + torch.erf(mf / math.sqrt(2))) + mf * torch.exp(-0.5 * mf * mf) / math.sqrt(2 * math.pi)
    assert rel_err(dm, (dy.float() @ w2.float().t()) * gelu_grad) < 1e-2


@pytest.mark.parametrize("T,h,with_res", [(1000, 256, True), (1001, 2048, True), (1003, 2048, False),
                                           (999, 4096, True), (517, 8192, True), (300, 264, False),
                                           (5, 512, True), (4099, 1024, False),
                                           # backward v5 at every ring width class (h = 256 * NV,
                                           # NV = 3, 6, 7) and fewer rows than SMs
                                           (777, 768, True), (20000, 1536, False), (2, 1792, True)])
def test_layernorm_fwd_bwd(T, h, with_res):
    # ragged row counts, h up to 8192 and h % 256 != 0, with and without the
    # residual gradient; dgain / dbias accumulate into their prior contents
    x = rnd(T, h, seed=13) * 2 + 0.5
    gain = (1 + 0.1 * torch.randn(h, device=DEV))
    bias = 0.1 * torch.randn(h, device=DEV)
    y = K.layernorm(x, gain, bias)
    xf = x.float().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xf, (h,), gain, bias, eps=1e-5)
    dy = rnd(T, h, seed=14)
    dres = rnd(T, h, seed=15) if with_res else None
    dg0, db0 = torch.randn(h, device=DEV), torch.randn(h, device=DEV)
    dg, db = dg0.clone(), db0.clone()
    dx = torch.empty_like(x)
    K.layernorm_bwd(dy, x, gain, dres, dx, dg, db)
    torch.cuda.synchronize()
    assert rel_err(y, ref) < 1e-2
    (gx,) = torch.autograd.grad(ref, xf, dy.float())
    xhat = (xf - xf.mean(-1, keepdim=True)) / torch.sqrt(xf.var(-1, unbiased=False, keepdim=True) + 1e-5)
    want_dx = gx + dres.float() if with_res else gx
    assert rel_err(dx, want_dx) < 2e-2
    assert rel_err(dg - dg0, (dy.float() * xhat).sum(0)) < 1e-3
    assert rel_err(db - db0, dy.float().sum(0)) < 1e-3


def attn_ref(qkv, s, b, heads):
    """fp32 causal attention on [s*b, 3h] -> (o [s*b, h], lse [b, heads, s])."""
    h = qkv.shape[1] // 3
    d = h // heads
    t = qkv.float().view(s, b, 3, heads, d).permute(2, 1, 3, 0, 4)  # [3, b, n, s, d]
    q, k, v = t[0], t[1], t[2]
    sc = q @ k.transpose(-1, -2) / math.sqrt(d)
    mask = torch.triu(torch.ones(s, s, dtype=torch.bool, device=DEV), 1)
    sc = sc.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(sc, -1)
    o = torch.softmax(sc, -1) @ v  # [b, n, s, d]
    return o.permute(2, 0, 1, 3).reshape(s * b, h), lse


ATTN_CASES = [(256, 1, 2, 64), (384, 1, 2, 128), (200, 2, 2, 64), (1024, 1, 4, 128), (130, 1, 1, 128),
              # multi-head 1-D grids in longest-first order, ragged tails
              (2048, 2, 3, 128), (1000, 1, 8, 64)]


@pytest.mark.parametrize("s,b,heads,d", ATTN_CASES)
def test_attention_forward(s, b, heads, d):
    h = heads * d
    qkv = rnd(s * b, 3 * h, seed=16)
    o = torch.empty(s * b, h, dtype=torch.bfloat16, device=DEV)
    lse = torch.empty(b, heads, s, device=DEV)
    K.attention_fwd(qkv, s, b, heads, o, lse)
    torch.cuda.synchronize()
    o_ref, lse_ref = attn_ref(qkv, s, b, heads)
    assert rel_err(o, o_ref) < 2e-2
    assert (lse - lse_ref).abs().max().item() < 2e-2


@pytest.mark.parametrize("s,b,heads,d", ATTN_CASES)
def test_attention_backward(s, b, heads, d):
    h = heads * d
    qkv = rnd(s * b, 3 * h, seed=17)
    o = torch.empty(s * b, h, dtype=torch.bfloat16, device=DEV)
    lse = torch.empty(b, heads, s, device=DEV)
    K.attention_fwd(qkv, s, b, heads, o, lse)
    d_o = rnd(s * b, h, seed=18)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(b * heads * s, device=DEV)
    dq_ws = K.attention_bwd_ws(s, b, heads, d, DEV)
    K.attention_bwd(qkv, o, d_o, lse, s, b, heads, dqkv, delta, dq_ws)
    torch.cuda.synchronize()
    qf = qkv.float().requires_grad_(True)
    o_ref, _ = attn_ref(qf, s, b, heads)
    (g,) = torch.autograd.grad(o_ref, qf, d_o.float())
    for part in range(3):
        sl = slice(part * h, (part + 1) * h)
        assert rel_err(dqkv[:, sl], g[:, sl]) < 3e-2, part


def test_gemm_rejects_unaligned_stride():
    # documented constraint: TMA needs 16-byte row strides (ld % 8 for bf16)
    x, dy = rnd(72, 300, seed=5), rnd(72, 200, seed=6)
    acc = torch.zeros(300, 200, device=DEV)
    with pytest.raises(K._lib.KernelLibraryError, match="HX_E_SHAPE"):
        K.linear_dw(x, dy, acc)


def test_mse_loss_and_axpy():
    z = rnd(4096, 256, seed=19)
    dz = torch.empty_like(z)
    slot = torch.zeros(1, dtype=torch.float64, device=DEV)
    K.mse_loss(z, dz, slot)
    y = torch.randn(1000, device=DEV)
    x = torch.randn(1000, device=DEV)
    want = y + x
    K.axpy(y, x)
    torch.cuda.synchronize()
    zf = z.double()
    assert abs(slot.item() / z.numel() - (zf * zf).mean().item()) < 1e-5 * (zf * zf).mean().item()
    assert rel_err(dz, z.float() * (2.0 / z.numel())) < 1e-2
    assert torch.allclose(y, want)


def test_kernel_timers_count_launches_per_entry_point():
    # bench.py's in-step roofline: every C-ABI call bracketed by CUDA events
    from paper_2507_00394_b200.runtime import _lib
    x, w = rnd(512, 256, seed=20), rnd(256, 512, scale=256 ** -0.5, seed=21)
    y = torch.empty(512, 512, dtype=torch.bfloat16, device=DEV)
    _lib.start_kernel_timers()
    for _ in range(3):
        K.linear(x, w, y)
    K.layernorm(x, torch.ones(256, device=DEV), torch.zeros(256, device=DEV))
    t = _lib.stop_kernel_timers()
    assert t["hx_gemm"]["launches"] == 3 and t["hx_ln_fwd"]["launches"] == 1
    assert all(v["total_ms"] > 0 and v["mean_ms"] == pytest.approx(v["total_ms"] / v["launches"])
               for v in t.values())
    # disabled again: no timers collected
    K.linear(x, w, y)
    assert _lib.stop_kernel_timers() == {}
