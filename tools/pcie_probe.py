import torch, time
x = torch.empty(524288000 // 8, dtype=torch.complex64).pin_memory()
d = torch.empty_like(x, device="cuda")
for _ in range(2): d.copy_(x, non_blocking=True); x.copy_(d, non_blocking=True)
torch.cuda.synchronize()
for name, f in [("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))]:
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); [f() for _ in range(5)]; e.record(); torch.cuda.synchronize()
    print(name, 5*524288000/ (s.elapsed_time(e)*1e-3)/1e9, "GB/s")
