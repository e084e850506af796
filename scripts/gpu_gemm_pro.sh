mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_refcontext.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 600 python bench.py --config suite --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_suite.log 2>&1
tail -n 5 gpurun_out/pytest_gemm.log
tail -n 1 gpurun_out/bench_suite.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['per_kernel_gbs']); print(d.get('per_kernel_ms'))"
