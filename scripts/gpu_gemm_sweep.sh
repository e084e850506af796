for g in 4 8 16 32; do for kc in 16 32; do
  v=$(FMB200_GEMM_GROUP_M=$g FMB200_GEMM_KC=$kc timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('check',{}).get('max_rel_err_all_entries_vs_exact_f64_kernel'))")
  echo "group_m $g kc $kc: $v"
done; done
