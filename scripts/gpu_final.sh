# end-of-round measurement pass on the final code (outputs in gpurun_out/r02f)
O=gpurun_out/r02f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
for c in c4r suite; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_default.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $O/launches_default.log 2>&1
timeout 2000 python scripts/ncu_round.py $O ${NCU_CAPS:-ncu_c3_copy ncu_suite_sigmoid ncu_suite_gelu ncu_suite_expr3} > $O/ncu_round.log 2>&1
tail -n 2 $O/pytest_gpu.log; tail -n 2 $O/smoke.log
for f in $O/bench*.log; do echo "== $f"; tail -n 1 $f | cut -c1-200; done
