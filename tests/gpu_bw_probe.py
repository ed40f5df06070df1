import torch, time
x = torch.empty(1<<27, dtype=torch.float64, device='cuda')  # 1 GiB
y = torch.empty_like(x)
def t(f, n=10):
    f(); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    best=1e9
    for _ in range(n):
        a.record(); f(); b.record(); torch.cuda.synchronize(); best=min(best,a.elapsed_time(b))
    return best
ms=t(lambda: x.zero_()); print("memset 1GiB", ms, "ms", x.numel()*8/ms/1e6, "GB/s")
ms=t(lambda: x.fill_(1.5)); print("fill   1GiB", ms, "ms", x.numel()*8/ms/1e6, "GB/s")
ms=t(lambda: y.copy_(x)); print("copy   1GiB", ms, "ms", 2*x.numel()*8/ms/1e6, "GB/s (r+w)")
ms=t(lambda: x.sum()); print("read   1GiB", ms, "ms", x.numel()*8/ms/1e6, "GB/s")
