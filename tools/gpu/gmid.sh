# iterations per CUDA-graph chunk at 64^3 (8 = product) and the transport at 64^3
V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))'
for i in 1 2; do for lib in default gm16 gm32 gm64; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_$lib.so; fi
  echo "$lib 64: $(python bench.py --n 64 --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "$V") T64: $(python bench.py --workload transport --n 64 --steps 600 2>/dev/null | python -c "$V") ens64: $(python bench.py --workload ensemble --n 64 --cells 8 --steps 200 2>/dev/null | python -c "$V")" >> gpurun_out/gmid.log
done; done
