# full GPU parity suite + smoke + suite bench (one call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config suite --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_suite.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log
tail -n 1 gpurun_out/bench_suite.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['per_kernel_gbs'])"
