"""Debug timeline of the tensor-core MLP adjoint's VJP kernel (CTA 0, stage 3,
first iteration) from a -DBODE_ADJ_PROF build: python tools/adj_prof.py LIB"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["BODE_LIB"] = sys.argv[1]
sys.argv = [sys.argv[0], "--config", "c4", "--reps", "1"]
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import adjoint_bench  # noqa: E402

try:
    adjoint_bench.main()
except SystemExit:
    pass
lib = ctypes.CDLL(os.environ["BODE_LIB"])
buf = (ctypes.c_longlong * 1024)()
n = lib.bode_debug_adj_prof(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(2, 256, 2)
for w, cnt in ((0, n // 1000), (1, n % 1000)):
    cnt = min(cnt, 256)
    t0 = a[w, 0, 1]
    print(f"thread {'0 (MMA)' if w == 0 else '128 (producer)'}: {cnt} stamps")
    prev = t0
    for k in range(min(cnt, 120)):
        tag, t = a[w, k]
        print(f"  tag {tag:3d}  t={t - t0:9d}  +{t - prev}")
        prev = t
