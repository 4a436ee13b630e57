# early PDL trigger sites (bit mask: 1 RS passes, 2 finalize, 4 RS-fix)
V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))'
for i in 1 2; do for lib in sel0 sel1 sel2 sel4 sel6; do
  export POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_$lib.so
  echo "$lib 64: $(python bench.py --n 64 --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "$V") 128: $(python bench.py --n 128 --steps 400 --no-cpu-baseline 2>/dev/null | python -c "$V") 256: $(python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "$V") ens128: $(python bench.py --workload ensemble --n 128 --steps 100 2>/dev/null | python -c "$V") T128: $(python bench.py --workload transport --n 128 --steps 300 2>/dev/null | python -c "$V")" >> gpurun_out/pdlsel2.log
done; done
