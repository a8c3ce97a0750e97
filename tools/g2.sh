timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --cpu-seconds 1 --no-e2e > gpurun_out/tm1.json 2> gpurun_out/tm1.err; tail -3 gpurun_out/tm1.err; cat gpurun_out/tm1.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['value'])"
