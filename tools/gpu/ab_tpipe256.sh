# transport 256^3: persistent axis-1 passes (POREFLOW_B200_M_PIPE=1) vs per-tile; Stokes 256^3 M pipe too
ST='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})'
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v["ms"],4) for k,v in d["stages"].items()})'
for i in 1 2; do for mp in 0 1; do
  echo "transport mpipe=$mp $(POREFLOW_B200_M_PIPE=$mp python bench.py --workload transport --n 256 --steps 200 2>/dev/null | python -c "$ST")" >> gpurun_out/tpipe256.log
  echo "stokes mpipe=$mp $(POREFLOW_B200_M_PIPE=$mp python bench.py --steps 200 --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/tpipe256.log
done; done
