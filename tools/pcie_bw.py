"""Pinned host<->device copy bandwidth on this box (context for bench.py's e2e leg)."""
import torch

dev = torch.device("cuda:0")
for mb in (48, 2560):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        print(f"{name} {mb} MB: {mb / 1024 / (ms / 1000):.1f} GiB/s")
    # both directions at once on two streams
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2 = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d2 = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    print(f"bidir {mb} MB each: {2 * mb / 1024 / (a.elapsed_time(b) / 1000):.1f} GiB/s total")
