import time, torch, numpy as np
n = 301**3
t = torch.randn(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
def tm(label, fn, reps=3):
    out=[]
    for _ in range(reps):
        torch.cuda.synchronize(); t0=time.perf_counter(); r=fn(); torch.cuda.synchronize(); out.append(time.perf_counter()-t0)
    print(f"{label:40s} " + " ".join(f"{x*1e3:7.1f}" for x in out) + " ms")
    return r
tm("pinned alloc (fresh, kept)", lambda: keep.append(torch.empty(n, dtype=torch.float64, pin_memory=True)) if (keep:=globals().setdefault('keep', [])) is not None else None)
tm("t.cpu() pageable", lambda: t.cpu())
def np_copy():
    a = np.empty(n); torch.from_numpy(a).copy_(t); return a
tm("copy_ into fresh numpy", np_copy)
buf = np.empty(n); buf[:] = 0
tm("copy_ into touched numpy", lambda: torch.from_numpy(buf).copy_(t))
p = torch.empty(n, dtype=torch.float64, pin_memory=True)
tm("copy_ into pinned (reused)", lambda: p.copy_(t))
tm("pinned copy + np.copy out", lambda: (p.copy_(t), p.numpy().copy()))
def np_empty_touch():
    a = np.empty(n); a[::512] = 0; return a
tm("np.empty + touch pages", np_empty_touch)
cr = torch.cuda.cudart()
def reg():
    a = np.empty(n)
    rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    torch.from_numpy(a).copy_(t)
    cr.cudaHostUnregister(a.ctypes.data)
    return a
tm("cudaHostRegister fresh numpy + copy", reg)
