#!/usr/bin/env python3
"""H2D bandwidth of the host-buffer entry points: r1_tensor_copy_from_host from
pinned and from pageable memory (staging lanes), and torch's own copy, for a
4 GB tensor.  Prints JSON lines."""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

ctx = r1.default_context()
L = _lib.lib()
n = 512 * 1024 * 1024  # 4 GiB of doubles
dims = (1024, 1024, 512)
t = r1.DeviceTensor.create(dims, ctx) if hasattr(r1.DeviceTensor, "create") else None
dev = torch.empty(n + 2, dtype=torch.float64, device="cuda")
t = r1.DeviceTensor.wrap(dev.data_ptr(), dims, ctx, keepalive=dev)
pinned = torch.empty(n, dtype=torch.float64, pin_memory=True)
pinned.fill_(1.0)
pageable = np.ones(n)
for name, ptr in (("pinned", pinned.data_ptr()), ("pageable", pageable.ctypes.data)):
    for _ in range(2):
        _lib.check(L.r1_tensor_copy_from_host(ctx.handle, t.handle, ctypes.cast(ptr, _lib._dp)))
    ctx.synchronize()
    reps = 4
    ts = time.perf_counter()
    for _ in range(reps):
        _lib.check(L.r1_tensor_copy_from_host(ctx.handle, t.handle, ctypes.cast(ptr, _lib._dp)))
    ctx.synchronize()
    dt = (time.perf_counter() - ts) / reps
    print(json.dumps({"source": name, "GB/s": round(8 * n / dt / 1e9, 2)}), flush=True)
ts = time.perf_counter()
for _ in range(4):
    dev[:n].copy_(pinned, non_blocking=True)
torch.cuda.synchronize()
print(json.dumps({"source": "torch pinned copy_", "GB/s": round(8 * n * 4 / (time.perf_counter() - ts) / 1e9, 2)}))
