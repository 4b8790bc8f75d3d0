# Round evidence: GPU tests, smoke, bench (default args), launch list, ncu --set full of both step
# kernels, FP32 FMA peak microbenchmark.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xy2?_(hh_)?kernel|zst4?_kernel" -s 10 -c 2 \
  -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
timeout 120 ./tools/microbench/fma_tput > gpurun_out/fma_tput.log 2>&1
timeout 600 python tools/sweep.py 512 > gpurun_out/sweep.log 2>&1
