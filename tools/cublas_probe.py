"""cuBLAS reference rates on the GPU box (torch.matmul): f64 DGEMM, TF32 and
bf16 at 8192^3 -- the library ceilings the hand-written GEMMs are compared to."""
import torch


def rate(dtype, n=8192, tf32=False, reps=5):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.rand(n, n, device="cuda", dtype=dtype)
    b = torch.rand(n, n, device="cuda", dtype=dtype)
    c = a @ b.t()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        c = a @ b.t()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return 2 * n ** 3 / best / 1e9


print("cuBLAS f64 DGEMM 8192^3: %.1f TF/s" % rate(torch.float64))
print("cuBLAS f32 (no TF32) 8192^3: %.1f TF/s" % rate(torch.float32))
print("cuBLAS TF32 8192^3: %.1f TF/s" % rate(torch.float32, tf32=True))
print("cuBLAS bf16 8192^3: %.1f TF/s" % rate(torch.bfloat16))
