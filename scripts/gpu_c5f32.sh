mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_refcontext.py tests/test_gpu_api.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 600 python bench.py --config c5f32 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5f32.log 2>&1
tail -n 5 gpurun_out/pytest_gemm.log
for f in gpurun_out/bench_c5f32.log; do echo "== $f"; tail -n 1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('check'), d.get('per_kernel_ms'))"; done
