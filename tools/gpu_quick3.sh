mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-parity > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline']['kernel_ms'], d['e2e']['value'], d['e2e']['pinned']['value'])"
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl 2>&1; cat gpurun_out/e2e_probe.jsonl
timeout 900 python tools/radius_sweep.py 3 4 5 6 > gpurun_out/radius_sweep.jsonl 2>&1; cat gpurun_out/radius_sweep.jsonl
bash tools/gpu_tests.sh
