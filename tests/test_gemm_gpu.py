"""tcgen05/TMA GEMM numerics vs a plain PyTorch fp32 reference (bf16 inputs)."""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _gemm(A, a_mn, B, b_mn, M, N, K, relu=0, out_f32=0, mask=None, bn=0):
    from paper_1909_11985_b200 import _lib
    L = _lib.lib()
    out = torch.empty(M, N, dtype=torch.float32 if out_f32 else torch.bfloat16, device="cuda")
    rc = L.edl_gemm_bf16(A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn,
                         out.data_ptr(), N, M, N, K, relu, out_f32,
                         mask.data_ptr() if mask is not None else None,
                         N if mask is not None else 0, bn,
                         C.c_void_p(torch.cuda.current_stream().cuda_stream))
    _lib.check(rc)
    torch.cuda.synchronize()
    return out


def _ref(A, a_mn, B, b_mn):
    a = A.float().t() if a_mn else A.float()
    b = B.float() if b_mn else B.float().t()
    return a @ b


# bn: 0 = auto (CTA-pair kernel when M >= 256), 1..256 = 1-SM kernel with that N tile,
# 1000 + x = CTA-pair (cta_group::2) kernel with N tile x, 2256 = CTA-pair kernel with 256-wide
# tiles split over K between two pairs (fp32 partials exchanged through DSMEM)
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K,bn", [(128, 128, 64, 128), (256, 256, 512, 0),
                                      (512, 4096, 4096, 0), (512, 4096, 4096, 128),
                                      (384, 448, 320, 112), (4096, 1024, 512, 256),
                                      (256, 256, 128, 1128), (512, 512, 256, 1256),
                                      (384, 320, 200, 1192), (4096, 1024, 512, 1128),
                                      (512, 4096, 4096, 1256), (512, 4096, 4096, 2256),
                                      (256, 256, 512, 2256), (384, 768, 1000, 2256),
                                      (512, 1024, 200, 2256)])
def test_gemm_layouts(a_mn, b_mn, M, N, K, bn):
    torch.manual_seed(0)
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(torch.bfloat16).cuda()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(torch.bfloat16).cuda()
    out = _gemm(A, a_mn, B, b_mn, M, N, K, out_f32=1, bn=bn)
    ref = _ref(A, a_mn, B, b_mn)
    err = (out - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-3 * scale + 1e-3, (err, scale)


@pytest.mark.parametrize("bn", [0, 128, 1128, 1256, 2256])
def test_gemm_relu_mask_bf16(bn):
    torch.manual_seed(1)
    M, N, K = 512, 1024, 768
    A = torch.randn(M, K).to(torch.bfloat16).cuda()
    B = torch.randn(N, K).to(torch.bfloat16).cuda()
    mask = torch.randn(M, N).to(torch.bfloat16).cuda()
    out = _gemm(A, 0, B, 0, M, N, K, relu=1, mask=mask, bn=bn)
    ref = torch.relu(_ref(A, 0, B, 0)) * (mask.float() > 0)
    assert torch.allclose(out.float(), ref.bfloat16().float(), rtol=2e-2, atol=2e-1)


@pytest.mark.parametrize("M,N,K", [(256, 128, 64), (1024, 1024, 512), (4096, 4096, 512),
                                   (384, 640, 192)])
def test_wgrad_sgd_fused(M, N, K):
    """dW = dY^T X fused with master -= scale * bf16(dW), W = bf16(master) (mlp.cu update)."""
    from paper_1909_11985_b200 import _lib
    L = _lib.lib()
    torch.manual_seed(2)
    dy = torch.randn(K, M).to(torch.bfloat16).cuda()
    x = torch.randn(K, N).to(torch.bfloat16).cuda()
    master = torch.randn(M, N, device="cuda")
    m0 = master.clone()
    W = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    scale = 1e-3
    rc = L.edl_gemm_wgrad_sgd(dy.data_ptr(), M, x.data_ptr(), N, master.data_ptr(), W.data_ptr(),
                              N, M, N, K, C.c_float(scale),
                              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    _lib.check(rc)
    torch.cuda.synchronize()
    g = (dy.float().t() @ x.float()).bfloat16().float()
    ref = m0 - scale * g
    # bf16 rounding of the fp32 accumulator can differ by 1 ulp where the sums differ in order
    tol = scale * g.abs().max().item() * 2 ** -7 + 1e-6
    assert (master - ref).abs().max().item() <= tol
    assert torch.equal(W, master.bfloat16())

