# MF_T as two launches (product) vs one (lib_nosplit)
timeout 900 python -m pytest tests/test_gpu_fused_transport.py tests/test_gpu_baseline_configs.py -x -q -p no:cacheprovider -k "transport or cfg2" > gpurun_out/tfsplit_pytest.log 2>&1; echo "exit $?" >> gpurun_out/tfsplit_pytest.log
ST='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v*1000,1) for k,v in d["stages_ms"].items()})'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_nosplit.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  for n in 256 128 64; do
  echo "$lib n=$n $(python bench.py --workload transport --n $n --steps 300 2>/dev/null | python -c "$ST")" >> gpurun_out/tfsplit.log
  done
done; done
