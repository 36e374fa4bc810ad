"""Kernel-level numerics on the B200: each sm_100a kernel against a plain PyTorch fp32
computation of the same op on the same (bf16-rounded) inputs."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2306_09342_b200 import kernels, _capi
    _capi.lib()
    torch.backends.cuda.matmul.allow_tf32 = False
    return kernels


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


def gelu_ref(u):
    c, a = 0.7978845608028654, 0.044715
    return 0.5 * u * (1 + torch.tanh(c * (u + a * u ** 3)))


def gelu_slope_ref(u):
    c, a = 0.7978845608028654, 0.044715
    t = torch.tanh(c * (u + a * u ** 3))
    return 0.5 * (1 + t) + 0.5 * u * (1 - t * t) * c * (1 + 3 * a * u * u)


# (M, N, K); N = 1664 / 384 end in a 128-column tile (the CTA pair's narrow N = 128 product)
SHAPES = [(296, 512, 200), (128, 256, 64), (1000, 768, 768), (264, 2304, 136), (304, 1664, 192),
          (200, 384, 128)]


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (0, 0), (1, 1), (1, 0)])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bn", [256, 128, 512], ids=["128x256", "128x128", "2sm-256x256"])
def test_gemm_majors_bf16(K, a_mn, b_mn, shape, bn):
    from paper_2306_09342_b200._capi import RP_EPI_BF16
    M, N, Kd = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + Kd)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    Bm = torch.randn(Kd, N, device="cuda", generator=g).bfloat16()
    Ast = A.t().contiguous() if a_mn else A
    Bst = Bm if b_mn else Bm.t().contiguous()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(Ast, Bst, M, N, Kd, a_mn=a_mn, b_mn=b_mn, epi=RP_EPI_BF16, out=out, bn=bn)
    ref = A.float() @ Bm.float()
    assert rel(out, ref) < 1e-2


def test_gemm_persistent_grid_independent(K):
    """Same bits whatever the CTA cap (what PaReprop's SM partitioning relies on)."""
    from paper_2306_09342_b200._capi import RP_EPI_F32
    M, N, Kd = 1024, 768, 4096
    A = torch.randn(Kd, M, device="cuda").bfloat16()
    Bm = torch.randn(Kd, N, device="cuda").bfloat16()
    outs = []
    for bn, cap in ((256, 0), (256, 5), (256, 37), (512, 0), (512, 6), (512, 38)):
        o = torch.empty(M, N, device="cuda")
        ws = torch.empty(4 * M * N, device="cuda")
        K.gemm(A, Bm, M, N, Kd, a_mn=1, b_mn=1, epi=RP_EPI_F32, out=o, splits=4, workspace=ws,
               max_ctas=cap, bn=bn)
        outs.append(o)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    assert torch.equal(outs[3], outs[4]) and torch.equal(outs[3], outs[5])
    ref = A.float().t() @ Bm.float()
    assert rel(outs[0], ref) < 1e-4


@pytest.mark.parametrize("bn", [256, 512])
@pytest.mark.parametrize("splits", [1, 3, 8])
@pytest.mark.parametrize("N", [768, 1664])
def test_gemm_wgrad_splitk(K, splits, bn, N):
    from paper_2306_09342_b200._capi import RP_EPI_F32
    T, M = 5000, 384
    X = torch.randn(T, M, device="cuda").bfloat16()
    dY = torch.randn(T, N, device="cuda").bfloat16()
    o = torch.empty(M, N, device="cuda")
    ws = torch.empty(splits * M * N, device="cuda")
    K.gemm(X, dY, M, N, T, a_mn=1, b_mn=1, epi=RP_EPI_F32, out=o, splits=splits, workspace=ws,
           bn=bn)
    ref = X.float().t() @ dY.float()
    assert rel(o, ref) < 1e-4


@pytest.mark.parametrize("bn", [256, 512])
@pytest.mark.parametrize("N", [1024, 1664])
def test_gemm_bias_gelu(K, bn, N):
    from paper_2306_09342_b200._capi import RP_EPI_BIAS_GELU
    M, Kd = 515, 192
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    W = (0.1 * torch.randn(Kd, N, device="cuda")).bfloat16()
    bias = torch.randn(N, device="cuda")
    a = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    u = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(A, W, M, N, Kd, a_mn=0, b_mn=1, epi=RP_EPI_BIAS_GELU, out=a, out2=u, bias=bias, bn=bn)
    uref = A.float() @ W.float() + bias
    assert rel(u, uref) < 1e-2
    assert rel(a, gelu_ref(uref)) < 1e-2


@pytest.mark.parametrize("bn", [256, 512])
@pytest.mark.parametrize("sign", [1.0, -1.0])
@pytest.mark.parametrize("Kd,N", [(3072, 768), (768, 768), (512, 320), (1664, 1664)])
def test_gemm_residual(K, sign, bn, Kd, N):
    """Residual epilogue; CTA-pair tiles with K <= 1024 store through TMA (ragged N too)."""
    from paper_2306_09342_b200._capi import RP_EPI_RESID
    M = 700
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    W = (0.05 * torch.randn(Kd, N, device="cuda")).bfloat16()
    bias = torch.randn(N, device="cuda")
    res = torch.randn(M, N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    K.gemm(A, W, M, N, Kd, a_mn=0, b_mn=1, epi=RP_EPI_RESID, out=out, aux=res, bias=bias,
           sign=sign, bn=bn)
    ref = res + sign * (A.float() @ W.float() + bias)
    assert rel(out, ref) < 1e-4
    # in place (out aliases the residual), as the inverse uses it
    res2 = res.clone()
    K.gemm(A, W, M, N, Kd, a_mn=0, b_mn=1, epi=RP_EPI_RESID, out=res2, aux=res2, bias=bias,
           sign=sign, bn=bn)
    assert torch.equal(res2, out)


@pytest.mark.parametrize("bn", [256, 512])
@pytest.mark.parametrize("N", [1024, 1664])
def test_gemm_gelu_slope_then_mul(K, bn, N):
    """Recompute epilogue keeps gelu'(u); the MLP dgrad multiplies by it (N = 1664: the CTA
    pair's last tile column is an N = 128 product; its column sums must stop at N)."""
    from paper_2306_09342_b200._capi import RP_EPI_BIAS_GELU_SLOPE, RP_EPI_MUL
    M, Kd = 600, 256
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    W = (0.1 * torch.randn(Kd, N, device="cuda")).bfloat16()
    bias = torch.randn(N, device="cuda")
    a = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    sl = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(A, W, M, N, Kd, a_mn=0, b_mn=1, epi=RP_EPI_BIAS_GELU_SLOPE, out=a, out2=sl, bias=bias,
           bn=bn)
    uref = A.float() @ W.float() + bias
    assert rel(a, gelu_ref(uref)) < 1e-2
    assert rel(sl, gelu_slope_ref(uref)) < 1e-2
    dY = torch.randn(M, 512, device="cuda").bfloat16()
    W2 = (0.05 * torch.randn(N, 512, device="cuda")).bfloat16()
    du = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    part = torch.empty((M + 31) // 32, N, device="cuda")
    K.gemm(dY, W2, M, N, 512, a_mn=0, b_mn=0, epi=RP_EPI_MUL, out=du, aux=sl, bn=bn,
           colsum_part=part)
    ref = (dY.float() @ W2.float().t()) * sl.float()
    assert rel(du, ref) < 1e-2
    # fused column sums of the fp32 product (the MLP hidden-bias gradient)
    cs = K.colsum_parts(part)
    assert rel(cs, ref.sum(0)) < 1e-4
    assert torch.equal(cs, K.colsum_parts(part))


@pytest.mark.parametrize("bn", [256, 512])
def test_gemm_gelu_bwd(K, bn):
    from paper_2306_09342_b200._capi import RP_EPI_GELU_BWD
    M, N, Kd = 640, 3072, 768
    dY = torch.randn(M, Kd, device="cuda").bfloat16()
    W2 = (0.05 * torch.randn(N, Kd, device="cuda")).bfloat16()  # W2 is [h, d] = [N][K]
    u = torch.randn(M, N, device="cuda").bfloat16()
    du = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(dY, W2, M, N, Kd, a_mn=0, b_mn=0, epi=RP_EPI_GELU_BWD, out=du, aux=u, bn=bn)
    ref = (dY.float() @ W2.float().t()) * gelu_slope_ref(u.float())
    assert rel(du, ref) < 1e-2


@pytest.mark.parametrize("rows,cols", [(1000, 768), (37, 192), (513, 1024), (64, 1664)])
def test_layer_norm_fwd_bwd(K, rows, cols):
    x = torch.randn(rows, cols, device="cuda") * 3 + 1
    gamma = torch.randn(cols, device="cuda")
    beta = torch.randn(cols, device="cuda")
    y, mean, rstd = K.layer_norm_fwd(x, gamma, beta, 1e-5)
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    xh = (x - mu) / torch.sqrt(var + 1e-5)
    assert rel(y, xh * gamma + beta) < 1e-2
    assert rel(rstd, 1 / torch.sqrt(var.squeeze(-1) + 1e-5)) < 1e-5
    dy = torch.randn(rows, cols, device="cuda").bfloat16()
    dres = torch.randn(rows, cols, device="cuda")
    dxb = torch.empty(rows, cols, device="cuda", dtype=torch.bfloat16)
    dx, dg, db = K.layer_norm_bwd(x, mean, rstd, gamma, dy, dres=dres, dx_bf16=dxb)
    g = dy.float() * gamma
    dx_ref = (g - g.mean(-1, keepdim=True) - xh * (g * xh).mean(-1, keepdim=True)) / torch.sqrt(
        var + 1e-5) + dres
    assert rel(dx, dx_ref) < 1e-4
    assert rel(dxb, dx_ref) < 1e-2
    assert rel(dg, (dy.float() * xh).sum(0)) < 1e-4
    assert rel(db, dy.float().sum(0)) < 1e-4
    # bit-reproducible
    dx2, dg2, db2 = K.layer_norm_bwd(x, mean, rstd, gamma, dy, dres=dres)
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2) and torch.equal(db, db2)
    # fused column sum of the produced cotangent (the next block's output-bias grad)
    cs = torch.empty(cols, device="cuda")
    dx3, dg3, db3 = K.layer_norm_bwd(x, mean, rstd, gamma, dy, dres=dres, dx_colsum=cs)
    assert torch.equal(dx, dx3) and torch.equal(dg, dg3) and torch.equal(db, db3)
    assert rel(cs, dx_ref.sum(0)) < 1e-4
    # the two-kernel path (row kernel + column pass) computes the same dx
    from paper_2306_09342_b200 import _capi
    _capi.lib().rp_set_ln_bwd_impl(0)
    try:
        dx4, dg4, db4 = K.layer_norm_bwd(x, mean, rstd, gamma, dy, dres=dres)
    finally:
        _capi.lib().rp_set_ln_bwd_impl(1)
    assert rel(dx4, dx) < 1e-6
    assert rel(dg4, dg) < 1e-5 and rel(db4, db) < 1e-5


@pytest.mark.parametrize("nparts,cols", [(1576, 3072), (788, 1536), (257, 40), (300, 100),
                                         (5000, 64), (129, 3072), (2, 8), (12544, 512),
                                         (2049, 200), (70000, 32)])
def test_colsum_parts(K, nparts, cols):
    """Many-part column sums (one cluster launch above 256 parts, one CTA per 32 columns
    below): fp64 reference, ragged part counts and column counts, accumulate, determinism."""
    part = torch.randn(nparts, cols, device="cuda")
    ref = part.double().sum(0)
    out = K.colsum_parts(part)
    assert (out.double() - ref).abs().max().item() < 1e-5 * nparts ** 0.5 * 4
    assert torch.equal(out, K.colsum_parts(part))
    base = torch.randn(cols, device="cuda")
    acc = base.clone()
    K.colsum_parts(part, out=acc, accumulate=True)
    assert torch.allclose(acc.double(), base.double() + ref, atol=1e-4 * nparts ** 0.5)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_colsum(K, dtype):
    x = torch.randn(50432 // 8, 3072, device="cuda").to(dtype)
    out = K.colsum(x)
    assert rel(out, x.float().sum(0)) < 1e-4
    assert torch.equal(out, K.colsum(x))


@pytest.mark.parametrize("B,N,H,hd", [(2, 197, 2, 104), (3, 64, 3, 32), (1, 130, 2, 128),
                                      (2, 50, 4, 96), (1, 300, 1, 104), (64, 49, 4, 32),
                                      (5, 49, 2, 16), (2, 100, 3, 24), (1, 700, 1, 32),
                                      (512, 49, 2, 32), (1000, 49, 1, 16), (300, 64, 2, 104),
                                      (3, 197, 3, 72), (2, 256, 2, 120), (1, 384, 1, 104),
                                      (4, 65, 2, 104), (1, 208, 16, 104)])
def test_attention_general_head_dim(K, B, N, H, hd):
    """head_dim != 64 (e.g. the G48 config's 104, Swin's 32 over 49-token windows) runs on
    the mma.sync kernels with the head padded to 32 / 64 / 128 columns in smem."""
    qkv = torch.randn(B * N, 3 * H * hd, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, N, H, head_dim=hd)
    qkv_r = qkv.float().requires_grad_(True)
    o_ref, lse_ref = attn_ref(qkv_r, B, N, H, hd)
    assert rel(out, o_ref) < 1e-2
    assert rel(lse / 1.4426950408889634, lse_ref) < 1e-4
    dout = torch.randn(B * N, H * hd, device="cuda").bfloat16()
    dqkv = K.attention_bwd(qkv, out, lse, dout, B, N, H, head_dim=hd)
    o_ref.backward(dout.float())
    g = qkv_r.grad
    for i, name in enumerate("qkv"):
        sl = slice(i * H * hd, (i + 1) * H * hd)
        assert rel(dqkv[:, sl], g[:, sl]) < 2e-2, name
    assert torch.equal(dqkv, K.attention_bwd(qkv, out, lse, dout, B, N, H, head_dim=hd))


def attn_ref(qkv, B, N, H, hd=64):
    q, k, v = qkv.float().view(B, N, 3, H, hd).permute(2, 0, 3, 1, 4)
    s = (q @ k.transpose(-1, -2)) / hd ** 0.5
    p = torch.softmax(s, -1)
    o = p @ v
    return o.permute(0, 2, 1, 3).reshape(B * N, H * hd), torch.logsumexp(s, -1)


@pytest.fixture(params=[0, 1, 2, 3], ids=["tcgen05", "mma_sync", "tcgen05_2pass", "tcgen05_dst"])
def impl(request):
    """The process-global attention implementation switch, restored whatever the test
    does (a failed assertion must not leave impl 1 / 2 active for later tests)."""
    from paper_2306_09342_b200 import _capi
    _capi.check(_capi.lib().rp_set_attention_impl(request.param), "set_attention_impl")
    try:
        yield request.param
    finally:
        _capi.lib().rp_set_attention_impl(0)


@pytest.mark.parametrize("B,N,H", [(64, 197, 12), (40, 208, 16), (96, 150, 8)])
def test_fused_attention_bwd_matches_dst_path(K, B, N, H):
    """The single-pass fused backward (impl 0, N <= 208) against the dS^T round-trip path
    (impl 3) at shapes with several (sequence, head) pairs per CTA: the same products in a
    different association, so they agree to bf16 rounding, and each is deterministic."""
    from paper_2306_09342_b200 import _capi
    qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, N, H)
    dout = torch.randn(B * N, H * 64, device="cuda").bfloat16()
    res = {}
    try:
        for impl in (0, 3):
            _capi.check(_capi.lib().rp_set_attention_impl(impl), "set_attention_impl")
            a = K.attention_bwd(qkv, out, lse, dout, B, N, H)
            assert torch.equal(a, K.attention_bwd(qkv, out, lse, dout, B, N, H))
            res[impl] = a.float()
    finally:
        _capi.lib().rp_set_attention_impl(0)
    assert rel(res[0], res[3]) < 1e-2


@pytest.mark.parametrize("B,N,H", [(4, 197, 12), (3, 208, 2), (2, 192, 3), (2, 160, 2),
                                   (3, 17, 2), (2, 33, 1), (1, 100, 3), (2, 224, 2)])
def test_attention_fwd_split_pv(K, B, N, H):
    """Forward variant 0 (P V split by key half over two issuers, N <= 208) against the
    single-issuer ping-pong kernel (variant 2) and the fp32 reference: the same P, two
    partial accumulators summed in the epilogue, so O agrees to fp32 rounding (bf16 output),
    and the LSE is the same computation."""
    from paper_2306_09342_b200 import _capi
    torch.manual_seed(31 * N + B)
    qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
    res = {}
    try:
        for v in (0, 2):
            assert _capi.lib().rp_set_attention_fwd_variant(v) == 0
            res[v] = K.attention_fwd(qkv, B, N, H)
            assert all(torch.equal(a, b) for a, b in zip(res[v], K.attention_fwd(qkv, B, N, H)))
    finally:
        _capi.lib().rp_set_attention_fwd_variant(0)
    assert _capi.lib().rp_set_attention_fwd_variant(3) == 3  # RP_ERR_CONFIG
    o_ref, lse_ref = attn_ref(qkv.float(), B, N, H)
    assert rel(res[0][0], o_ref) < 1e-2
    assert (res[0][0].float() - res[2][0].float()).abs().max().item() <= 2 ** -7 * \
        res[2][0].float().abs().max().item()
    assert torch.equal(res[0][1], res[2][1])


@pytest.mark.parametrize("B,N,H,hd", [(64, 49, 4, 32), (600, 49, 3, 32), (7, 1, 2, 32),
                                      (9, 2, 3, 32), (5, 17, 2, 32), (4, 33, 2, 16),
                                      (3, 64, 2, 32), (6, 49, 2, 64), (3, 63, 1, 104),
                                      (200, 49, 2, 24), (1, 48, 1, 32)])
def test_attention_window_kernels(K, B, N, H, hd):
    """N <= 64 (Swin windows): the single-tile kernels (window variant 0, the default) against
    the fp32 reference and the general mma.sync kernels (variant 1)."""
    from paper_2306_09342_b200 import _capi
    torch.manual_seed(1000 * N + hd + B)
    qkv = torch.randn(B * N, 3 * H * hd, device="cuda").bfloat16()
    dout = torch.randn(B * N, H * hd, device="cuda").bfloat16()
    res = {}
    try:
        for v in (0, 1):
            assert _capi.lib().rp_set_attention_window_variant(v) == 0
            out, lse = K.attention_fwd(qkv, B, N, H, head_dim=hd)
            dq = K.attention_bwd(qkv, out, lse, dout, B, N, H, head_dim=hd)
            assert torch.equal(dq, K.attention_bwd(qkv, out, lse, dout, B, N, H, head_dim=hd))
            res[v] = (out, lse, dq)
    finally:
        _capi.lib().rp_set_attention_window_variant(0)
    assert _capi.lib().rp_set_attention_window_variant(2) == 3  # RP_ERR_CONFIG
    qkv_r = qkv.float().requires_grad_(True)
    o_ref, lse_ref = attn_ref(qkv_r, B, N, H, hd)
    o_ref.backward(dout.float())
    out, lse, dq = res[0]
    assert rel(out, o_ref) < 1e-2
    assert rel(lse / 1.4426950408889634, lse_ref) < 1e-4
    assert rel(out, res[1][0]) < 1e-2 and rel(lse, res[1][1]) < 1e-5
    g = qkv_r.grad
    for i, name in enumerate("qkv"):
        sl = slice(i * H * hd, (i + 1) * H * hd)
        if N == 1 and name != "v":  # no gradient wrt q, k: ours is rounding noise
            assert (dq[:, sl].float() - g[:, sl]).abs().max() < 1e-3 * g.abs().max(), name
        else:
            tol = 4e-2 if (N == 2 and name != "v") else 2e-2
            assert rel(dq[:, sl], g[:, sl]) < tol, name


def test_attention_impl_switch_validates():
    from paper_2306_09342_b200 import _capi
    assert _capi.lib().rp_set_attention_impl(4) == 3  # RP_ERR_CONFIG
    assert _capi.lib().rp_set_attention_impl(-1) == 3
    assert _capi.lib().rp_set_attention_impl(0) == 0


@pytest.mark.parametrize("B,N,H", [(2, 197, 12), (3, 64, 2), (1, 5, 1), (2, 512, 4), (1, 130, 3), (2, 300, 2), (1, 480, 3), (3, 768, 1),
                                   (3, 256, 2), (2, 129, 1), (3, 1, 2), (8, 2, 4), (1, 17, 1),
                                   (4, 257, 1), (3, 208, 5), (2, 128, 3), (1, 144, 2), (2, 200, 7),
                                   (300, 197, 1)])
def test_attention_fwd_bwd(K, B, N, H, impl):
    torch.manual_seed(7919 * B + 131 * N + H)  # inputs fixed per case (order-independent)
    qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, N, H)
    qkv_r = qkv.float().requires_grad_(True)
    o_ref, lse_ref = attn_ref(qkv_r, B, N, H)
    assert rel(out, o_ref) < 1e-2
    assert rel(lse / 1.4426950408889634, lse_ref) < 1e-4
    dout = torch.randn(B * N, H * 64, device="cuda").bfloat16()
    dqkv = K.attention_bwd(qkv, out, lse, dout, B, N, H)
    o_ref.backward(dout.float())
    g = qkv_r.grad
    for i, name in enumerate("qkv"):
        sl = slice(i * H * 64, (i + 1) * H * 64)
        if g[:, sl].abs().max() < 1e-6 * g.abs().max():
            # N = 1: softmax over one key has no gradient wrt q, k; ours is rounding noise
            # of dP - D, bounded relative to the whole gradient
            assert (dqkv[:, sl].float() - g[:, sl]).abs().max() < 1e-3 * g.abs().max(), name
        else:
            # N = 2, q and k only: dS of a row is (+x, -x), x = P0 (dP0 - D) = P0 P1 (dP0 - dP1)
            # evaluated as a cancellation against D = rowsum(dO * O) from the bf16-stored O
            # (the flash-style backward), then rounded to bf16 for the tensor core; dq =
            # x (k0 - k1) and dk carry that error undamped (2.6 % seen on unseeded inputs), so
            # they get 4 %; dv = P^T dO does not involve D and keeps 2 %. The case runs 64
            # query rows (B H N) so the max-relative metric is not decided by one row.
            tol = 4e-2 if (N == 2 and name != "v") else 2e-2
            assert rel(dqkv[:, sl], g[:, sl]) < tol, name
    assert torch.equal(dqkv, K.attention_bwd(qkv, out, lse, dout, B, N, H))


@pytest.mark.parametrize("bn", [256, 128, 512])
@pytest.mark.parametrize("H", [4, 26])
def test_gemm_rowdot(K, bn, H):
    """RP_EPI_ROWDOT: bf16 output plus, per (row, 64-column head), the dot of the bf16 output
    with aux -- the attention backward's D = rowsum(dO * O) laid out [(seq, head), token]
    (H = 26: N = 1664 ends in a 128-column tile)."""
    from paper_2306_09342_b200._capi import RP_EPI_ROWDOT
    S_, Ntok, Kd = 5, 197, 768
    M, N = S_ * Ntok, H * 64
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    W = (0.05 * torch.randn(N, Kd, device="cuda")).bfloat16()
    O = torch.randn(M, N, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    D = torch.full((S_ * H * Ntok,), float("nan"), device="cuda")
    K.gemm(A, W, M, N, Kd, a_mn=0, b_mn=0, epi=RP_EPI_ROWDOT, out=out, aux=O, rowdot=D,
           rd_seq=Ntok, bn=bn)
    ref = A.float() @ W.float().t()
    assert rel(out, ref) < 1e-2
    dref = (out.float() * O.float()).view(S_, Ntok, H, 64).sum(-1).permute(0, 2, 1).reshape(-1)
    assert rel(D, dref) < 1e-5
