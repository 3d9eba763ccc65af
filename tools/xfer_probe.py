"""Host<->device transfer probe: pageable vs pinned bandwidth, host memcpy
bandwidth, cudaHostRegister cost (sizes of the C2 e2e payload)."""
import os, time
import numpy as np, torch
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
os.system("lscpu | grep -E 'Model name|^CPU\\(s\\)|Thread|Socket|NUMA node\\(s\\)'")
dev = torch.device("cuda", 0)
N = 64 * 2**20
d = torch.empty(N, dtype=torch.uint8, device=dev)
pg = np.ones(N, np.uint8)
pn = torch.empty(N, dtype=torch.uint8, pin_memory=True); pn.fill_(1)
def t(f, k=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k
pgt = torch.from_numpy(pg)
for name, f in [("h2d pageable", lambda: d.copy_(pgt)), ("h2d pinned", lambda: d.copy_(pn, non_blocking=True)),
                ("d2h pageable", lambda: pgt.copy_(d)), ("d2h pinned", lambda: pn.copy_(d, non_blocking=True))]:
    s = t(f); print(f"{name}: {N/s/1e9:.1f} GB/s ({s*1e3:.2f} ms / 64 MiB)")
dst = np.empty_like(pg)
s = t(lambda: np.copyto(dst, pg)); print(f"np.copyto 1 thread: {N/s/1e9:.1f} GB/s")
for k in range(3):
    a = np.ones(N, np.uint8)
    t0 = time.perf_counter()
    r = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, N, 0)
    t1 = time.perf_counter()
    torch.cuda.cudart().cudaHostUnregister(a.ctypes.data)
    t2 = time.perf_counter()
    print(f"hostRegister 64MiB: {1e3*(t1-t0):.2f} ms, unregister {1e3*(t2-t1):.2f} ms rc={r}")

t0 = time.perf_counter(); x = torch.empty(N, dtype=torch.uint8, pin_memory=True); print(f"pinned alloc {1e3*(time.perf_counter()-t0):.2f} ms")
del x
t0 = time.perf_counter(); x = torch.empty(N, dtype=torch.uint8, pin_memory=True); print(f"pinned alloc (cached) {1e3*(time.perf_counter()-t0):.2f} ms")
