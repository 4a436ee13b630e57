timeout 900 python -m pytest tests/test_gpu_fused_transport.py tests/test_gpu_baseline_configs.py -x -q -p no:cacheprovider -k "transport or cfg2" > gpurun_out/r02an_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02an_pytest.log
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_tfboth0.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  for args in "--n 256" "--n 128"; do
  echo "$lib $args $(python bench.py --workload transport $args --steps 200 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})')" >> gpurun_out/r02an_ab.log
  done
done; done
