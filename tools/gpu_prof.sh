# ncu --set full capture of both step kernels (one GPU), 512^3 bench config.
mkdir -p gpurun_out
K=${1:-"xy2?_(hh_)?kernel|zst4?_kernel"}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 10 -c 2 -o gpurun_out/prof \
  python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
