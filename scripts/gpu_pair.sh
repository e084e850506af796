mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tiled.py -x -q > gpurun_out/pytest_tiled.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiled.log
timeout 300 python scripts/transpose_probe.py ${SIZES:-8192 10000} > gpurun_out/probe.log 2>&1
cap() {  # name regex
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s 0 -c 1 -o gpurun_out/$1 -f python scripts/transpose_probe.py 8192 > gpurun_out/$1.log 2>&1
ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1.details.csv 2>/dev/null
ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/$1.sass.csv.gz
rm -f gpurun_out/$1.ncu-rep
}
# cap ncu_pair8k 'k_copy_pair'
cap ncu_pair8k_expr2 'k_copy_pair.*Log.*float'
tail -3 gpurun_out/pytest_tiled.log; cat gpurun_out/probe.log
