# GPU pass 3: full tests + smoke, bench, e2e probe, radius sweep, parity report,
# initcheck, ncu launch list + full capture of both hot kernels.
mkdir -p gpurun_out
bash tools/gpu_tests.sh
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline']['kernel_ms'], d['e2e']['value'])"
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl 2>&1; cat gpurun_out/e2e_probe.jsonl
timeout 900 python tools/radius_sweep.py 3 4.5 5.5 6 6.5 7 8 9 > gpurun_out/radius_sweep.jsonl 2>&1; cat gpurun_out/radius_sweep.jsonl
timeout 900 python tools/parity_report.py > gpurun_out/parity.txt 2>&1; tail -4 gpurun_out/parity.txt
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 50 python tools/sanitize_case.py > gpurun_out/sanitize_initcheck.log 2>&1; tail -3 gpurun_out/sanitize_initcheck.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"zst4|xy2" -s 6 -c 2 -o gpurun_out/prof python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
ls gpurun_out
