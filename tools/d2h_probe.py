import time, numpy as np, torch
n = 33554432
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d.fill_(3); torch.cuda.synchronize()
def t(f, k=5):
    best = 1e9
    for _ in range(k):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - a)
    return round(best * 1e3, 3)
def pageable():
    out = np.empty(n, np.uint8); torch.from_numpy(out).copy_(d)
bounce = torch.empty(n, dtype=torch.uint8, pin_memory=True)
def bounce_copy():
    out = np.empty(n, np.uint8); bounce.copy_(d); out[:] = bounce.numpy()
keep = []
def fresh_pinned():
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.copy_(d); keep.append(h)
print("pageable", t(pageable), "bounce+memcpy", t(bounce_copy), "fresh pinned", t(fresh_pinned))
