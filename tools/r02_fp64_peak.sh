#!/bin/bash
# FP64 peak re-measured with the SM clock sampled during the runs (the 37.04 TF
# denominator had no clock record).  20 back-to-back runs of tools/fp64_peak, then a sustained
# cuBLAS DGEMM loop; nvidia-smi every 100 ms meanwhile.
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 100 > gpurun_out/fp64_clocks.csv &
SMI=$!
for i in $(seq 20); do ./tools/fp64_peak; done > gpurun_out/fp64_peak_runs.txt 2>&1
python - <<'PY' >> gpurun_out/fp64_peak_runs.txt 2>&1
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2): torch.matmul(a, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 0; e0.record(); t0 = time.time()
while time.time() - t0 < 4.0:
    torch.matmul(a, b); n += 1
e1.record(); torch.cuda.synchronize()
print(f"cuBLAS DGEMM 8192^3 sustained {n} calls: {2*8192**3*n/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s")
PY
kill $SMI
