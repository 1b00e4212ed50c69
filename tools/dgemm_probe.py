import torch, json
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for (B, n) in [(32, 512), (128, 128), (8, 2048), (1, 8192)]:
    a = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(B, n, n + 1, dtype=torch.float64, device="cuda")
    for _ in range(3): c = torch.bmm(a, b)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        s.record(); c = torch.bmm(a, b); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
    res[f"{B}x{n}"] = {"ms": best, "tflops": 2 * B * n * n * (n + 1) / best / 1e9}
print(json.dumps(res))
