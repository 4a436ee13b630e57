timeout 900 python -m pytest tests/test_gpu_fused_transport.py tests/test_gpu_baseline_configs.py -x -q -p no:cacheprovider > gpurun_out/r02ad_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02ad_pytest.log
POREFLOW_B200_M_PIPE=1 timeout 900 python -m pytest tests/test_gpu_fused_transport.py -x -q -p no:cacheprovider >> gpurun_out/r02ad_pytest.log 2>&1; echo "exit256 $?" >> gpurun_out/r02ad_pytest.log
for i in 1 2; do for mp in 0 1; do
  for args in "--n 128" "--n 128 --tcells 3" "--n 256"; do
    echo "mpipe=$mp $args $(POREFLOW_B200_M_PIPE=$mp python bench.py --workload transport $args --steps 200 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})')" >> gpurun_out/r02ad_ab.log
  done
done; done
