"""Measured dense INT8 tensor-core throughput on this GPU: cuBLASLt (torch._int_mm)
int8 x int8 -> int32 at 8192^3, best of 10 (burst) and back to back for 2 s
(sustained), CUDA events. The evidence behind the INT8 peak bench.py divides by."""
import json
import time

import torch


def main(n=8192):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cnt = 0
    t_end = time.perf_counter() + 2.0
    s.record()
    while time.perf_counter() < t_end:
        for _ in range(10):
            torch._int_mm(a, b)
        cnt += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    sus = s.elapsed_time(e) / cnt
    ops = 2.0 * n ** 3
    print(json.dumps(dict(what="cuBLASLt int8 GEMM (torch._int_mm) %d^3" % n, burst_ms=best,
                          burst_tops=ops / best / 1e9, sustained_ms=sus, sustained_tops=ops / sus / 1e9,
                          gpu=torch.cuda.get_device_name())))


if __name__ == "__main__":
    main()
