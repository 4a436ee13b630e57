# RS_T register-resident (k_trs_w) vs k_trs at 256^3: transport tests, then A/B bench
timeout 900 python -m pytest tests/test_gpu_fused_transport.py tests/test_gpu_steps.py -x -q -p no:cacheprovider > gpurun_out/trsw_pytest.log 2>&1; echo "exit $?" >> gpurun_out/trsw_pytest.log
for i in 1 2; do for tw in 1 0; do
  export POREFLOW_B200_TRS_W=$tw
  echo "trs_w=$tw $(python bench.py --workload transport --n 256 --steps 200 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})')" >> gpurun_out/trsw_ab.log
done; done
