import torch
x = torch.empty(921_600_000, dtype=torch.uint8, device="cuda").fill_(1)
f = x.view(torch.float32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, fn in [("sum f32", lambda: f.sum()), ("amax f32", lambda: f.amax()), ("copy", lambda: y.copy_(x))]:
    if name == "copy":
        y = torch.empty_like(x)
    ts = []
    for k in range(6):
        flush.zero_(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if k >= 2: ts.append(s.elapsed_time(e))
    ms = min(ts)
    b = 921.6e6 * (2 if name == "copy" else 1)
    print(f"{name}: {ms*1e3:.1f} us  {b/ms/1e6:.0f} GB/s")
