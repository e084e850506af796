mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gemm.log
timeout 300 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_c5.log
if [ -n "$NCU" ]; then bash scripts/ncu_capture.sh c5_gemm k_gemm 0 -- python bench.py --config c5 --steps 1 --warmup 0 --no-e2e --no-cpu; fi
tail -n 30 gpurun_out/pytest_gemm.log; tail -n 3 gpurun_out/bench_c5.log
