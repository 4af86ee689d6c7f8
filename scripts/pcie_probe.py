"""Host<->device copy bandwidth on the GPU box: one pinned 3.3 GB buffer (the
cfg 4 particle state) copied H2D and D2H as one copy, or split into chunks
issued round-robin on 2 or 4 streams (separate copy engines). GPU only:
    python scripts/pcie_probe.py
"""
import time

import torch


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    nbytes = 3_288_334_336
    n = nbytes // 8
    host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    host.fill_(1.0)
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        chunks = 4 * ns if ns > 1 else 1
        step = (n + chunks - 1) // chunks

        def h2d():
            for c in range(chunks):
                with torch.cuda.stream(streams[c % ns]):
                    dev[c * step:(c + 1) * step].copy_(host[c * step:(c + 1) * step], non_blocking=True)

        def d2h():
            for c in range(chunks):
                with torch.cuda.stream(streams[c % ns]):
                    host[c * step:(c + 1) * step].copy_(dev[c * step:(c + 1) * step], non_blocking=True)

        th, td = timed(h2d), timed(d2h)
        print(f"streams {ns} chunks {chunks}: H2D {nbytes / th / 1e9:.1f} GB/s ({th * 1e3:.1f} ms), "
              f"D2H {nbytes / td / 1e9:.1f} GB/s ({td * 1e3:.1f} ms)", flush=True)


if __name__ == "__main__":
    main()
