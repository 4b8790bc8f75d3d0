# Round-end evidence pass (one B200): tests + smoke, bench lines, sanitizers,
# ncu launch list + full capture, parity report.  Logs under gpurun_out/.
mkdir -p gpurun_out
bash tools/gpu_tests.sh
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --mode strong-cfg4 --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --gpus 2 --share-gpu --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/bench_n2share.json 2> gpurun_out/bench_n2share.err
bash tools/sanitize.sh
timeout 900 python tools/parity_report.py > gpurun_out/parity.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"zst4|xy2" -s 6 -c 2 -o gpurun_out/prof python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline']['kernel_ms'], d['e2e']['value'])"
ls gpurun_out
