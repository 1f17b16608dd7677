"""D2H options for the stored values g (3x2160x3840 f32): sparse + host scatter
(current), dense pageable, dense into a cached pinned block."""
import time, torch, numpy as np
C, H, W = 3, 2160, 3840
g = torch.zeros(C, H, W, device="cuda")
sup = torch.rand(H, W, device="cuda") < 0.05
g[:, sup] = torch.rand(C, int(sup.sum()), device="cuda")
torch.cuda.synchronize()
def sparse():
    idx = torch.nonzero(sup.reshape(-1)).squeeze(1)
    vals = g.reshape(C, -1)[:, idx]
    out = np.zeros((C, H, W), np.float32)
    out.reshape(C, -1)[:, idx.cpu().numpy()] = vals.cpu().numpy()
    return out
def dense_pageable():
    return g.cpu().numpy()
def dense_pinned():
    out = torch.empty((C, H, W), dtype=torch.float32, pin_memory=True)
    out.copy_(g)
    return out.numpy()
for fn in (sparse, dense_pageable, dense_pinned, sparse, dense_pageable, dense_pinned):
    keep = None
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t = time.perf_counter()
        keep = fn()
        ts.append(time.perf_counter() - t)
    print(fn.__name__, [round(x * 1e3, 1) for x in ts], flush=True)
