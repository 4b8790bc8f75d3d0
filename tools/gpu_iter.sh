# Iteration: GPU tests, smoke, sweep, then an ncu capture of the given kernel regex.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/sweep.py 512 > gpurun_out/sweep.log 2>&1
if [ -n "$1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s 10 -c 1 -o gpurun_out/prof \
  python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
fi
