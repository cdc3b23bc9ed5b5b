"""H2D / D2H bandwidth: one stream vs split across streams, and both directions at once."""
import torch
dev = torch.device("cuda", 0)
N = 16 << 20
x = torch.empty(N, dtype=torch.uint8).pin_memory()
y = torch.empty(N, dtype=torch.uint8, device=dev)
x2 = torch.empty(N, dtype=torch.uint8).pin_memory()
y2 = torch.empty(N, dtype=torch.uint8, device=dev)
ss = [torch.cuda.Stream() for _ in range(4)]
def timeit(f, reps=20):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    for s in ss: torch.cuda.current_stream().wait_stream(s)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def split(dst, src, k):
    cur = torch.cuda.current_stream()
    n = dst.numel() // k
    for i in range(k):
        ss[i].wait_stream(cur)
        with torch.cuda.stream(ss[i]):
            dst[i * n:(i + 1) * n].copy_(src[i * n:(i + 1) * n], non_blocking=True)
for k in (1, 2, 4):
    ms = timeit(lambda: split(y, x, k))
    print(f"h2d split {k}: {N / ms / 1e6:.1f} GB/s")
    ms = timeit(lambda: split(x, y, k))
    print(f"d2h split {k}: {N / ms / 1e6:.1f} GB/s")
def both():
    cur = torch.cuda.current_stream()
    ss[0].wait_stream(cur); ss[1].wait_stream(cur)
    with torch.cuda.stream(ss[0]): y.copy_(x, non_blocking=True)
    with torch.cuda.stream(ss[1]): x2.copy_(y2, non_blocking=True)
ms = timeit(both)
print(f"bidirectional: {N / ms / 1e6:.1f} GB/s each way")
