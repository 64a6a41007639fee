"""Host<->device copy rates for one 301^3 fp64 field (218 MB): pageable vs
pinned H2D, pinned D2H, and the host-side memcpy into pinned staging."""
import time
import numpy as np
import torch

n = 301 ** 3
a = np.random.default_rng(0).standard_normal(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
pin.copy_(torch.from_numpy(a))
torch.cuda.synchronize()


def t(fn, reps=5):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return float(np.median(out))


gb = n * 8 / 1e9
res = {
    "h2d_pageable": gb / t(lambda: d.copy_(torch.from_numpy(a))),
    "h2d_pinned": gb / t(lambda: d.copy_(pin, non_blocking=True)),
    "d2h_pinned": gb / t(lambda: pin.copy_(d, non_blocking=True)),
    "host_copy_into_pinned_torch": gb / t(lambda: pin.copy_(torch.from_numpy(a))),
    "host_copy_into_pinned_numpy": gb / t(lambda: np.copyto(pin.numpy(), a)),
    "torch_threads": torch.get_num_threads(),
}

# both directions at once (the pipelined host->host step overlaps them):
# seconds for one field each way, on two copy streams
d2 = torch.empty_like(d)
pin2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s_in):
        d.copy_(pin, non_blocking=True)
    with torch.cuda.stream(s_out):
        pin2.copy_(d2, non_blocking=True)
    s_in.synchronize()
    s_out.synchronize()


res["bidirectional_each_way"] = gb / t(both)
print({k: round(v, 2) if isinstance(v, float) else v for k, v in res.items()}, "GB/s")
