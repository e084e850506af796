mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
for c in ${CONFIGS:-c1 c2 c3 c4}; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; done
for spec in $NCU; do IFS=: read name kre cfg <<< "$spec"; bash scripts/ncu_capture.sh $name $kre 0 -- python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu; done
tail -n 3 gpurun_out/pytest_gpu.log
for f in gpurun_out/bench*.log; do echo "== $f"; tail -n 1 $f | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:800]); continue
    print(d['value'], d['ms_per_step'], d['roofline']['per_kernel_gbs'], d.get('check'))"; done
