# RS_T: u / H straight into registers (product: 4-row tiles at 256) vs staged (lib_ureg0) vs 2-row tiles (lib_uregr2)
timeout 900 python -m pytest tests/test_gpu_fused_transport.py tests/test_gpu_baseline_configs.py -x -q -p no:cacheprovider -k "transport or cfg2" > gpurun_out/ureg_pytest.log 2>&1; echo "exit $?" >> gpurun_out/ureg_pytest.log
ST='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_ureg0.so paper_2312_15554_b200/build/lib_uregr2.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  for n in 256 128; do
  echo "$lib n=$n $(python bench.py --workload transport --n $n --steps 200 2>/dev/null | python -c "$ST")" >> gpurun_out/ureg_ab.log
  done
done; done
