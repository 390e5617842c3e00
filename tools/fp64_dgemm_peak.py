"""cuBLAS DGEMM peak (torch.matmul fp64, 8192^3), burst and 4 s sustained -- the FP64 roofline denominator.

Mirrors MEASURED_PEAKS.json's bf16 method (best of 10 burst; back-to-back for 4 s sustained) so the
FP64 figure is measured the same way as the driver's bf16/HBM peaks.
"""
import json
import time

import torch


def main(n: int = 8192) -> None:
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2.0 * n ** 3 / (best * 1e-3) / 1e12
    count = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b)
        count += 1
        if count % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sustained = count * 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(json.dumps({"op": "cublas_dgemm", "n": n, "burst_tflops": round(burst, 3),
                      "sustained_tflops": round(sustained, 3)}))


if __name__ == "__main__":
    main()
