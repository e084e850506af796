mkdir -p gpurun_out
cap() {  # name regex
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s 0 -c 1 -o gpurun_out/$1 -f python bench.py --config suite --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/$1.log 2>&1
ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1.details.csv 2>/dev/null
ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/$1.sass.csv.gz
rm -f gpurun_out/$1.ncu-rep
}
cap ncu_gelu 'Tanh'
cap ncu_expr3 'Div.*Log<Mul<Log'
cap ncu_swish 'Div<In<0>, SAdd<0, Exp'
