#!/bin/bash
# One GPU session: bench line (+ reference arm), plain run + ncu launch list of one bench step, full ncu capture
# of the two hot kernels (INT8-sliced contraction + tiled Newton update) on a fixed cfg-2 workload, and of the cfg-3 Newton
# kernel on a 4096-sample cfg-3 workload.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
P="python tools/profile_case.py 2 65536"
$P > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"oz_gemm_kernel" -s 2 -c 1 -o gpurun_out/full $P > gpurun_out/ncu_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"newton_tgj" -s 2 -c 1 -o gpurun_out/full_lu $P > gpurun_out/ncu_full_lu.log 2>&1
P3="python tools/profile_case.py 3 4096"
$P3 > gpurun_out/plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"newton_tgh" -s 2 -c 1 -o gpurun_out/full_lu3 $P3 > gpurun_out/ncu_full_lu3.log 2>&1
for f in gpurun_out/ncu_full.log gpurun_out/ncu_full_lu.log gpurun_out/ncu_full_lu3.log; do tail -n 2 $f; done
# offline projection kernel: throughput line + one full capture
python tools/projection_perf.py 100 262144 > gpurun_out/projection_perf.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"project_convection" -s 3 -c 1 -o gpurun_out/full_proj python tools/projection_perf.py 100 65536 > gpurun_out/ncu_proj.log 2>&1
