# finalize shape at 64^3 / 128^3: threads (1024 / 512) and running sums per thread (4 / 2 / 8)
V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))'
for i in 1 2; do for lib in default f512 u2 u8 f512u2; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_$lib.so; fi
  echo "$lib 64: $(python bench.py --n 64 --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "$V") 128: $(python bench.py --n 128 --steps 400 --no-cpu-baseline 2>/dev/null | python -c "$V") T64: $(python bench.py --workload transport --n 64 --steps 600 2>/dev/null | python -c "$V")" >> gpurun_out/finv.log
done; done
