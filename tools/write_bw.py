"""Write-only and copy bandwidth of large buffers (torch fill_ / copy_), CUDA events, for the
projection's write roofline at output sizes beyond L2."""
import torch
dev = torch.device("cuda:0")
for mb in (40, 250, 1000, 4000):
    n = mb * 1000 * 1000 // 4
    x = torch.empty(n, dtype=torch.int32, device=dev)
    y = torch.empty(n, dtype=torch.int32, device=dev)
    for name, fn, b in (("fill", lambda: x.fill_(7), 4 * n), ("copy", lambda: y.copy_(x), 8 * n)):
        for _ in range(3):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) / reps
        print(f"{name} {mb:5d} MB  {t*1e3:9.1f} us  {b / t / 1e6:7.0f} GB/s")
    del x, y
