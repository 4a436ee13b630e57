SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v["ms"],4) for k,v in d["stages"].items()})'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_rs5.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --steps 200 --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/rs5.log
done; done
