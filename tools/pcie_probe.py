#!/usr/bin/env python
"""Host<->device copy ceiling for the bench's e2e leg: pinned H2D, D2H and
both directions concurrently on two streams, at the bench's per-step bytes
(538 MB each way).  Profiling aid; prints one JSON line."""
import json

import torch


def main(nbytes=537919488, reps=5):
    dev = torch.device("cuda", 0)
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn):
        fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize(dev)
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) * 1e-3 / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        torch.cuda.current_stream(dev).wait_stream(s1)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        torch.cuda.current_stream(dev).wait_stream(s2)

    def both():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        torch.cuda.current_stream(dev).wait_stream(s1)
        torch.cuda.current_stream(dev).wait_stream(s2)

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"bytes_each_way": nbytes, "h2d_GBps": nbytes / t1 / 1e9,
                      "d2h_GBps": nbytes / t2 / 1e9, "concurrent_ms": t3 * 1e3,
                      "concurrent_GBps_each_way": nbytes / t3 / 1e9}))


if __name__ == "__main__":
    main()
