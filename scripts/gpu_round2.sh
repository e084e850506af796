# round-2 measurement pass: tests, smoke, every bench config, reference arm,
# launch list of the default bench, ncu captures of every dominant kernel
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r02/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02/smoke.log
timeout 900 python bench.py > gpurun_out/r02/bench_default.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r02/bench_reference.log 2>&1
for c in c4r suite; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02/bench_$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02/launches_default.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/r02/launches_default.log 2>&1
timeout 3000 python scripts/ncu_round.py gpurun_out/r02 > gpurun_out/r02/ncu_round.log 2>&1
tail -n 3 gpurun_out/r02/pytest_gpu.log; tail -n 2 gpurun_out/r02/smoke.log
for f in gpurun_out/r02/bench*.log; do echo "== $f"; tail -n 1 $f | cut -c1-400; done
