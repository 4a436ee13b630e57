# persistent pipelined PK (k_pk_pipe, POREFLOW_B200_PK_PIPE=1) at 128^3: single cell and the 16-cell ensemble
V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))'
timeout 600 env POREFLOW_B200_PK_PIPE=1 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider -k "128" > gpurun_out/pkp128_pytest.log 2>&1; echo "exit $?" >> gpurun_out/pkp128_pytest.log
for i in 1 2; do for pp in 0 1; do
  echo "pk_pipe=$pp single128: $(POREFLOW_B200_PK_PIPE=$pp python bench.py --n 128 --steps 400 --no-cpu-baseline 2>/dev/null | python -c "$V") ens128: $(POREFLOW_B200_PK_PIPE=$pp python bench.py --workload ensemble --n 128 --steps 100 2>/dev/null | python -c "$V")" >> gpurun_out/pkp128.log
done; done
