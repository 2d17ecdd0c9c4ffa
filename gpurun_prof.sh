python -m pytest tests/test_parity_gpu.py -x -q -k "c1_64" 2>&1 | tail -1 > gpurun_out/pytest.log
MPB_SWEEP_NT=256 python -m pytest tests/test_parity_gpu.py -x -q -k "c1_64" 2>&1 | tail -1 >> gpurun_out/pytest.log
run() { env $1 python bench.py --steps 50 --warmup 3 --no-cpu $2 > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1 $2', round(d['value'],2), round(d['ms_per_step'],3), round(r['kernel_ms_per_step'],3), round(r['frac'],3))"; }
run X=1
run MPB_SWEEP_NT=256
run "MPB_SWEEP_NT=256 MPB_SWEEP_WAVES=32"
run "MPB_SWEEP_NT=256 MPB_SWEEP_T=448"
run X=1
cat gpurun_out/pytest.log
