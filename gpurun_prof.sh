MPB_ZWALL=kernel python -m pytest tests/test_parity_gpu.py tests/test_slab_gpu.py -x -q 2>&1 | tail -1 > gpurun_out/pytest.log
run() { env $1 python bench.py --steps 50 --warmup 3 --no-cpu $2 > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1 $2', round(d['value'],2), round(d['ms_per_step'],3), round(r['kernel_ms_per_step'],3), round(r['frac'],3))"; }
run X=1
run MPB_ZWALL=kernel
run X=1
run MPB_ZWALL=kernel
cat gpurun_out/pytest.log
