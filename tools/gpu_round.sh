# One GPU pass: pytest -m gpu + smoke, bench (N=1), reference arm, a strong
# cfg4 line at N=1 and a 2-rank shared-GPU line; logs under gpurun_out/.
mkdir -p gpurun_out
bash tools/gpu_tests.sh "$@"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --mode strong-cfg4 --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --gpus 2 --share-gpu --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/bench_n2share.json 2> gpurun_out/bench_n2share.err
tail -c 1500 gpurun_out/bench.json
