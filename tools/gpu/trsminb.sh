ST='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_trs5.so paper_2312_15554_b200/build/lib_trs6.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --workload transport --n 256 --steps 200 2>/dev/null | python -c "$ST")" >> gpurun_out/trsminb.log
done; done
