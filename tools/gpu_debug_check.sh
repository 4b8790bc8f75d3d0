# Debug-build check: the bounded-wait library (make debug) passes the parity
# suite; plus the plain-C caller and a sustained 200-step bench line.
mkdir -p gpurun_out
RSFG_LIB=paper_2404_02813_b200/lib/debug/librsfg.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x > gpurun_out/pytest_debuglib.log 2>&1; tail -2 gpurun_out/pytest_debuglib.log
RSFG_LIB=paper_2404_02813_b200/lib/debug/librsfg.so python tools/radius_sweep.py --steps 50 3 > gpurun_out/debuglib_speed.jsonl 2>&1; cat gpurun_out/debuglib_speed.jsonl
timeout 300 python -m pytest tests/test_abi.py -m gpu -q > gpurun_out/pytest_cabi.log 2>&1; tail -2 gpurun_out/pytest_cabi.log
timeout 900 python bench.py --steps 200 --warmup 10 --no-parity > gpurun_out/bench_200.json 2> gpurun_out/bench_200.err
python -c "import json; d=json.load(open('gpurun_out/bench_200.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'])"
