# ncu --set full capture of one kernel; exports raw + details CSV next to it
# usage: bash scripts/ncu_capture.sh <name> <kernel-regex> <launch-skip> -- <command...>
set -u
name=$1; kre=$2; skip=$3; shift 4
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c 1 \
    -o gpurun_out/$name -f "$@" > gpurun_out/$name.ncu.log 2>&1
ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>/dev/null
sz=$(stat -c %s gpurun_out/$name.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -gt 8000000 ]; then rm -f gpurun_out/$name.ncu-rep; fi
gzip -f gpurun_out/$name.sass.csv
