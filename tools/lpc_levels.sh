for v in 2,2,2 2,2,4 2,4,4 2,4,2 2,1,1 2,1,2; do GMG_LPC_LEVELS=$v python bench.py --no-next1 --no-cpu-baseline --steps 100 > gpurun_out/lpc_$v.json 2>/dev/null; done; echo done
