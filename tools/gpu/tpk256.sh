ST='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v*1000,1) for k,v in d["stages_ms"].items()})'
for i in 1 2; do for lib in default tpk5 tpk5np tpk3; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_$lib.so; fi
  echo "$lib $(python bench.py --workload transport --n 256 --steps 200 2>/dev/null | python -c "$ST")" >> gpurun_out/tpk256.log
done; done
