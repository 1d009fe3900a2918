"""H2D bandwidth probe: one 1.2 MB pinned copy vs split across streams, and a
zero-copy kernel read of mapped pinned memory."""
import torch
t = torch.rand(480, 640).pin_memory()
dev = torch.empty_like(t, device="cuda")
flat_t, flat_d = t.view(-1), dev.view(-1)
streams = [torch.cuda.Stream() for _ in range(4)]
def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
print("single copy ms", timed(lambda: dev.copy_(t, non_blocking=True)))
for k in (2, 4):
    n = flat_t.numel() // k
    def split():
        cur = torch.cuda.current_stream()
        ev = []
        for i in range(k):
            s = streams[i]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                flat_d[i * n:(i + 1) * n].copy_(flat_t[i * n:(i + 1) * n], non_blocking=True)
            e = torch.cuda.Event(); e.record(s); ev.append(e)
        for e in ev:
            cur.wait_event(e)
    print(f"split {k} ms", timed(split))
big = torch.rand(16, 480, 640).pin_memory()
bd = torch.empty_like(big, device="cuda")
print("19.7 MB copy ms", timed(lambda: bd.copy_(big, non_blocking=True)), "-> GB/s", 19.66e6 / timed(lambda: bd.copy_(big, non_blocking=True)) / 1e6)
