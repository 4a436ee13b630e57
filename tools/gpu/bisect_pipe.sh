for env in "X=1" "POREFLOW_B200_M_PIPE=0" "POREFLOW_B200_RSFIX_TMA=0" "POREFLOW_B200_M_PIPE=0 POREFLOW_B200_RSFIX_TMA=0"; do
  echo "== $env $(env $env python bench.py --workload pipeline --n 128 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["stokes_iterations"], d["transport_iterations"])')" >> gpurun_out/r02aw.log
done
