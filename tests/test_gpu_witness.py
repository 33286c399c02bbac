"""Witness generation on the GPU: the exact int16 x int16 -> int64 GEMM
(csrc/igemm.cu, byte-sliced mma.sync s8/u8) that produces the LoRA block's
wide products, against exact integer references."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2508_21393_b200 import device as D  # noqa: E402


@pytest.mark.parametrize("M,K,N", [(3, 5, 7), (130, 33, 70), (128, 64, 64), (1, 4096, 1),
                                   (256, (1 << 14) + 96, 72), (64, 1, 4096)])
def test_igemm16_exact_odd_shapes(M, K, N):
    g = torch.Generator().manual_seed(M * 7 + K + N)
    a = torch.randint(-2 ** 15, 2 ** 15, (M, K), generator=g, dtype=torch.int64)
    b = torch.randint(-2 ** 15, 2 ** 15, (K, N), generator=g, dtype=torch.int64)
    a[0, : min(K, 8)] = -32768  # extremes: the most negative high byte
    b[: min(K, 8), 0] = -32768
    if M > 1 and K > 1:
        a[1, 1] = 32767
    got = D.igemm16(a.to(torch.int16).cuda(), b.to(torch.int16).cuda()).cpu()
    want = a @ b  # exact int64 on the CPU
    assert torch.equal(got, want)


def test_igemm16_llama_shape_matches_fp64():
    """2048 x 4096 x 4096 (the X W products of a block): equal to the float64
    GEMM, which is exact here (|partial sums| < 2^42 < 2^53)."""
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randint(-2 ** 15, 2 ** 15, (2048, 4096), device="cuda", generator=g,
                      dtype=torch.int32).to(torch.int16)
    b = torch.randint(-2 ** 15, 2 ** 15, (4096, 4096), device="cuda", generator=g,
                      dtype=torch.int32).to(torch.int16)
    got = D.igemm16(a, b)
    want = torch.matmul(a.double(), b.double()).round_().long()
    assert torch.equal(got, want)


@pytest.mark.parametrize("M,K,N", [(2048, 4096, 16), (16, 2048, 4096), (4096, 2048, 16),
                                   (128, 33000, 64)])
def test_igemm16_split_k_skinny(M, K, N):
    """Skinny products (the LoRA-rank GEMMs of a block and of cfg2's witness)
    run split-K, the partial sums added into the output with 64-bit atomics:
    still exact (checked against int64 products on the CPU)."""
    g = torch.Generator().manual_seed(M + K + N)
    a = torch.randint(-2 ** 15, 2 ** 15, (M, K), generator=g, dtype=torch.int64)
    b = torch.randint(-2 ** 15, 2 ** 15, (K, N), generator=g, dtype=torch.int64)
    a[:, 0] = -32768
    b[0, :] = -32768
    got = D.igemm16(a.to(torch.int16).cuda(), b.to(torch.int16).cuda()).cpu()
    assert torch.equal(got, a @ b)


@pytest.mark.parametrize("lib", [True, False])
@pytest.mark.parametrize("M,K,N", [(2048, 4096, 1024), (1032, 8200, 520)])
def test_igemm16_library_and_kernel_paths(lib, M, K, N, monkeypatch):
    """Both product paths on the same shapes: the library int8 GEMM on byte
    planes (zkl_split_i16 + torch._int_mm + zkl_igemm_combine) and the repo's
    mma.sync kernel, each exact against int64 products."""
    monkeypatch.setattr(D, "IGEMM_LIB", lib)
    g = torch.Generator().manual_seed(M * 3 + K + N)
    a = torch.randint(-2 ** 15, 2 ** 15, (M, K), generator=g, dtype=torch.int64)
    b = torch.randint(-2 ** 15, 2 ** 15, (K, N), generator=g, dtype=torch.int64)
    a[0, :] = -32768
    a[1, :] = 32767
    b[:, 0] = -32768
    b[:, 1] = 32767
    got = D.igemm16(a.to(torch.int16).cuda(), b.to(torch.int16).cuda()).cpu()
    assert torch.equal(got, a @ b)
