python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
python bench.py --config c2 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
