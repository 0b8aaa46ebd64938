#!/usr/bin/env python
"""Host<->device copy rates from pinned memory (the e2e path's bound):
contiguous H2D / D2H, both directions at once, and row-strided 2-D copies
(column panels of a row-major matrix).  Prints one JSON line."""
import json
import torch


def rate(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


def main():
    nb = 1 << 30
    h = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
    h2 = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
    d = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
    d2 = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
    out = {}
    out["h2d_GBps"] = rate(lambda: d.copy_(h, non_blocking=True), nb)
    out["d2h_GBps"] = rate(lambda: h.copy_(d, non_blocking=True), nb)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    out["duplex_total_GBps"] = rate(both, 2 * nb)
    # column panels of a 16384 x 16384 fp32 matrix: 16384 rows of w floats, pitch 64 KiB
    H = h.view(16384, 16384)
    D = d.view(16384, 16384)
    for w in (512, 1024, 2048, 4096):
        out[f"h2d_2d_w{w}_GBps"] = rate(lambda: D[:, :w].copy_(H[:, :w], non_blocking=True), 16384 * w * 4)
    from cuda.bindings import runtime as rt
    st = torch.cuda.current_stream().cuda_stream
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
    for w in (1024, 2048, 4096):
        out[f"h2d_memcpy2d_w{w}_GBps"] = rate(lambda: rt.cudaMemcpy2DAsync(
            D.data_ptr(), 65536, H.data_ptr(), 65536, w * 4, 16384, H2D, st), 16384 * w * 4)
        out[f"d2h_memcpy2d_w{w}_h2048_GBps"] = rate(lambda: rt.cudaMemcpy2DAsync(
            H.data_ptr(), 65536, D.data_ptr(), 65536, w * 4, 2048, D2H, st), 2048 * w * 4, reps=20)
    for chunk in (16 << 20, 64 << 20, 128 << 20):
        k = chunk // 4
        out[f"h2d_chunk{chunk >> 20}MiB_GBps"] = rate(lambda: d[:k].copy_(h[:k], non_blocking=True), chunk, reps=20)
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
