#!/usr/bin/env python
"""FP32 roofline calibration on the GPU: FFMA and FFMA2 throughput and the
full-mask interaction rate (Table 2 analogue).  Prints one JSON line."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_06231_b200 import _lib  # noqa: E402


def timed(mode, blocks, threads, iters, reps=5):
    L = _lib.load()
    out = torch.zeros(1, device="cuda")
    s = torch.cuda.current_stream()
    st = ctypes.c_void_p(s.cuda_stream)
    assert L.sph_calibrate(mode, blocks, threads, iters, ctypes.c_void_p(out.data_ptr()), st) == 0
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sph_calibrate(mode, blocks, threads, iters, ctypes.c_void_p(out.data_ptr()), st)
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


def main():
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    res = {"sm_count": sm}
    for occ in (4, 8):
        blocks, threads = sm * occ, 256
        it = 2000
        t = timed(0, blocks, threads, it)
        res[f"ffma_tflops_occ{occ}"] = 2 * 64 * it * blocks * threads / t / 1e12
        t = timed(1, blocks, threads, it)
        res[f"ffma2_tflops_occ{occ}"] = 4 * 64 * it * blocks * threads / t / 1e12
    blocks, threads, it = sm * 8, 256, 40
    t = timed(2, blocks, threads, it)
    res["fullmask_interactions_per_s"] = 256 * it * blocks * threads / t
    res["fullmask_tflops_48"] = res["fullmask_interactions_per_s"] * 48 / 1e12
    t = timed(3, blocks, threads, it)                    # the production packed body (interact2)
    res["fullmask_packed_interactions_per_s"] = 256 * it * blocks * threads / t
    res["fullmask_packed_tflops_48"] = res["fullmask_packed_interactions_per_s"] * 48 / 1e12
    print(json.dumps(res))


if __name__ == "__main__":
    main()
