for pr in 0 64 128 256; do echo "== promo $pr"; FMB200_PAIR_PROMO=$pr timeout 300 python scripts/transpose_probe.py 8192 10000; done > gpurun_out/probe_promo.log 2>&1
cat gpurun_out/probe_promo.log
