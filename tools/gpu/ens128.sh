# 128^3 ensemble: cells per GPU and graph chunk length (lib_g8: 8 iterations per chunk)
V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))'
for i in 1 2; do
for lib in default paper_2312_15554_b200/build/lib_g8.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  for c in 8 16; do
    echo "$lib cells=$c $(python bench.py --workload ensemble --n 128 --cells $c --steps 200 2>/dev/null | python -c "$V")" >> gpurun_out/ens128.log
  done
  echo "$lib single128 $(python bench.py --n 128 --steps 400 --no-cpu-baseline 2>/dev/null | python -c "$V")" >> gpurun_out/ens128.log
done; done
