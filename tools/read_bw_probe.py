"""Read-bandwidth ceiling probe for the B = 1 stage-1 scan: how fast can
this box stream 3.072 GB (config B fp32 rows) with library kernels?
torch.sum over the rows, cuBLAS sgemv (rows @ q), and a bf16 gemv.
Prints GB/s per op (CUDA events, median of 20, after warm-up)."""
import torch

N, D = 1_000_000, 768


def bench(fn, nbytes, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    return ms, nbytes / (ms / 1e3) / 1e9


x = torch.randn(N, D, device="cuda")
q = torch.randn(D, device="cuda")
xb = x.to(torch.bfloat16)
qb = q.to(torch.bfloat16)
out = {}
out["sum_f32"] = bench(lambda: x.sum(), x.numel() * 4)
out["sgemv"] = bench(lambda: torch.mv(x, q), x.numel() * 4)
out["sgemm_n8"] = bench(lambda: x @ torch.randn(D, 8, device="cuda"), x.numel() * 4)
out["bf16_gemv"] = bench(lambda: torch.mv(xb, qb), xb.numel() * 2)
out["sum_bf16"] = bench(lambda: xb.sum(), xb.numel() * 2)
out["copy_f32_rw"] = bench(lambda: x.clone(), x.numel() * 8)
for k, (ms, gbs) in out.items():
    print(f"{k:12s} {ms * 1e3:9.1f} us {gbs:8.1f} GB/s")
