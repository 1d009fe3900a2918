import torch, time, ctypes as C, numpy as np
t = torch.rand(480, 640).pin_memory()
print("is_pinned", t.is_pinned())
dev = torch.empty_like(t, device="cuda")
for k in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dev.copy_(t, non_blocking=True); e1.record(); e1.synchronize()
    print("pinned H2D 1.2MB ms", e0.elapsed_time(e1))
a = t.numpy()
print("numpy ptr == tensor ptr", a.ctypes.data == t.data_ptr())
c = np.ascontiguousarray(a, dtype=np.float32)
print("ascontig same", c.ctypes.data == t.data_ptr())
p = np.random.rand(480, 640).astype(np.float32)
tp = torch.from_numpy(p)
for k in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0=time.perf_counter()
    e0.record(); dev.copy_(tp, non_blocking=True); e1.record(); e1.synchronize()
    print("pageable H2D 1.2MB ms", e0.elapsed_time(e1), "wall", (time.perf_counter()-t0)*1e3)
