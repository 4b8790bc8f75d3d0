# GPU pass 2: new tests, bench, radius sweep, sanitizers, ncu launch list + full capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_terms.py tests/test_gpu_parity.py tests/test_bench_launch.py tests/test_cpp_wrapper.py -m gpu -q -rf > gpurun_out/pytest_sub.log 2>&1; tail -3 gpurun_out/pytest_sub.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e'])"
timeout 600 python tools/radius_sweep.py > gpurun_out/radius_sweep.jsonl 2>&1; cat gpurun_out/radius_sweep.jsonl
bash tools/sanitize.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"zst4|xy2" -s 6 -c 2 -o gpurun_out/prof python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
