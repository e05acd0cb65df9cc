import os
import sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2302_03245_b200 import _lib
_lib.context()
n = 1 << 20
for trial in range(3):
    t = time.perf_counter(); a = _lib.pinned_empty(n); t1 = time.perf_counter()
    print(f"alloc fresh {1e3*(t1-t):.3f} ms")
prev = None
for i in range(6):
    t = time.perf_counter(); cur = _lib.pinned_empty(n); t1 = time.perf_counter()
    prev = cur
    print(f"alloc with previous alive->released {1e3*(t1-t):.3f} ms")
t = time.perf_counter(); x = np.empty(n); x[:] = 0; print(f"np.empty+touch {1e3*(time.perf_counter()-t):.3f} ms")
