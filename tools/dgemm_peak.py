"""cuBLAS DGEMM/ZGEMM ceiling via torch.matmul (comparator for the FP64 roofline)."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
props = torch.cuda.get_device_properties(0)
print(json.dumps({"gpu": props.name, "sms": props.multi_processor_count, "mem_gb": props.total_memory / 1e9}))
for dt, n, mult in [(torch.float64, 8192, 2), (torch.complex128, 4096, 8)]:
    a = torch.randn(n, n, dtype=dt, device=dev); b = torch.randn(n, n, dtype=dt, device=dev)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"kind": "cublas_" + str(dt), "n": n, "ms": ms, "tflops": mult * n**3 / ms / 1e9}))
