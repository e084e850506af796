mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "row_stats" > gpurun_out/pytest_c4r.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c4r.log
for pe in 6 4 2; do FMB200_ROW_SPLITS_PER_SM=$pe timeout 600 python bench.py --config c4r --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4r_$pe.log 2>&1; done
tail -2 gpurun_out/pytest_c4r.log
for f in gpurun_out/bench_c4r_*.log; do echo "== $f"; tail -n 1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('check'))"; done
