"""Dense-attention reference points on this B200 (library kernels, NOT part of the
product): torch SDPA (cuDNN and flash backends) and flashinfer if importable, at the
c2 attention shape (12 heads x 4680 queries x 4680 keys x d128, bf16) -- how far a
production Blackwell kernel gets on the same work as attn_fwd_v7 (1068 TFLOP/s)."""
import torch
import torch.nn.functional as F

H, L, d = 12, 4680, 128
q = torch.randn(1, H, L, d, device="cuda", dtype=torch.bfloat16)
k = torch.randn(1, H, L, d, device="cuda", dtype=torch.bfloat16)
v = torch.randn(1, H, L, d, device="cuda", dtype=torch.bfloat16)
flops = 4.0 * H * L * L * d


def bench(fn, name, reps=50):
    try:
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        print(f"{name:40s} {us:8.1f} us  {flops / us / 1e6:7.0f} TFLOP/s")
    except Exception as ex:  # noqa: BLE001
        print(f"{name:40s} unavailable: {type(ex).__name__}: {str(ex)[:100]}")


from torch.nn.attention import SDPBackend, sdpa_kernel
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
    def f(be=be):
        with sdpa_kernel(be):
            return F.scaled_dot_product_attention(q, k, v)
    bench(f, f"torch sdpa {be.name}")
try:
    import flashinfer
    qf, kf, vf = (t[0].transpose(0, 1).contiguous() for t in (q, k, v))  # [L, H, d]
    for backend in ("auto", "cutlass", "fa2", "trtllm-gen"):
        def g(backend=backend):
            return flashinfer.single_prefill_with_kv_cache(qf, kf, vf, causal=False, backend=backend)
        bench(g, f"flashinfer single_prefill {backend}")
except Exception as ex:  # noqa: BLE001
    print("flashinfer unavailable:", type(ex).__name__, str(ex)[:120])
