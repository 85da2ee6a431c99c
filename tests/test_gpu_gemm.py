"""The hand-written tcgen05 GEMM of the device decoder (st_gemm: C (op)= A W,
fused epilogues) against an fp32 PyTorch reference of the same op on the same
rounded inputs. Tolerance: the f16/bf16 rounding of the output (relative 2^-10
/ 2^-7 of the reference's magnitude) plus fp32 summation-order differences."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    return _capi


def gelu(x):
    return 0.5 * x * (1 + torch.erf(x / 2 ** 0.5))


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M,N,K,Z,epi", [
    (2048, 4096, 4096, 1, "store"),
    (300, 264, 256, 1, "store"),          # ragged M and N (tails of both tiles)
    (256, 4096, 1024, 3, "store"),        # batched Q|K|V over one activation
    (512, 16384, 1024, 1, "gelu"),
    (777, 1024, 4096, 1, "add_to"),
    (130, 32000, 512, 1, "store_f32"),    # LM-head shape (V=32000 = 125 tiles)
    (64, 264, 136, 1, "store_f32"),       # K not a multiple of the 64-deep K block
])
def test_gemm_matches_fp32(capi, dtype, M, N, K, Z, epi):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(dtype)
    w = (torch.randn(Z, K, N, device="cuda", generator=g) * K ** -0.5).to(dtype)
    ref = torch.einsum("mk,zkn->zmn", a.float(), w.float())
    out_dt = torch.float32 if epi == "store_f32" else dtype
    c0 = (torch.randn(Z, M, N, device="cuda", generator=g)).to(out_dt)
    out = c0.clone()
    if epi == "gelu":
        ref = gelu(ref)
    if epi == "add_to":
        ref = ref + c0.float()
    capi.gemm(a, w[0] if Z == 1 else w, out=out[0] if Z == 1 else out, epilogue=epi)
    torch.cuda.synchronize()
    got = out.float()
    eps = {torch.float16: 2 ** -10, torch.bfloat16: 2 ** -7, torch.float32: 2 ** -20}[out_dt]
    err = (got - ref).abs()
    tol = 2 * eps * ref.abs() + 1e-3 * ref.abs().max()
    assert bool((err <= tol).all()), f"max err {err.max().item():.3e} (ref max {ref.abs().max().item():.3e})"
