"""Pinned host -> device copy rate of 1 GB with 1 / 2 / 4 concurrent streams
(decides whether HostStepPipeline should spread a chunk's H2D over several
copy streams).  usage: python tools/micro/h2d_probe.py"""
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cur = torch.cuda.current_stream()
        step = n // ns
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"streams {ns} rep {rep}: {ms:.2f} ms  {n / ms / 1e6:.1f} GB/s")
