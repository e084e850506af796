# One GPU round: parity tests, smoke, every bench config (with CPU baseline +
# e2e), the reference arm, the ncu launch list of the default bench and ncu
# --set full captures of the top kernels.  Everything lands in gpurun_out/.
#   NCU="name:kernel-regex:config:skip ..."   (optional --set full captures)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
for c in ${CONFIGS:-c1 c3 c4 c4r c5 c5f32 suite}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.log 2>&1
done
if [ -z "$NO_LAUNCHES" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_default.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/launches_default.log 2>&1
fi
for spec in $NCU; do
  IFS=: read name kre cfg skip <<< "$spec"
  bash scripts/ncu_capture.sh $name $kre ${skip:-0} -- python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu
done
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log
for f in gpurun_out/bench*.log; do echo "== $f"; tail -n 1 $f | cut -c1-1500; done
