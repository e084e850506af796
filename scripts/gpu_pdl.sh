mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "not every_column" > gpurun_out/r02b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02b/pytest.log
timeout 900 python bench.py > gpurun_out/r02b/bench_default.log 2>&1
FMB200_PDL=0 timeout 900 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02b/bench_c1_nopdl.log 2>&1
FMB200_PDL=0 timeout 900 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02b/bench_c2_nopdl.log 2>&1
timeout 1800 python scripts/ncu_round.py gpurun_out/r02b ncu_c1_copy ncu_c2_accu_f32 ncu_c2_norm_f32 ncu_c2_accu_f64 ncu_c2_norm_f64 ncu_suite_expr1 > gpurun_out/r02b/ncu_round.log 2>&1
tail -n 4 gpurun_out/r02b/pytest.log
for f in gpurun_out/r02b/bench*.log; do echo "== $f"; tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['roofline'].get('per_kernel_gbs'))
for k,c in (d.get('configs') or {}).items(): print('  ',k, c.get('value'), c.get('ms_per_step'), c['roofline'].get('per_kernel_gbs'))"; done
