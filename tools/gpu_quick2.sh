mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_spec.py -m gpu -q -rf -x > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-parity > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline']['kernel_ms'], d['e2e']['value'], d['e2e']['pinned']['value'])"
timeout 900 python tools/radius_sweep.py 3 4 4.5 5 5.5 6 7 8 > gpurun_out/radius_sweep.jsonl 2>&1; cat gpurun_out/radius_sweep.jsonl
