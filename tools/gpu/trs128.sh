# RS_T tile rows at 128^3: 4 (product) vs 2 rows (64 threads; 4 or 6 CTAs/SM)
timeout 900 python -m pytest tests/test_gpu_fused_transport.py -x -q -p no:cacheprovider > gpurun_out/trs128_pytest.log 2>&1; echo "exit $?" >> gpurun_out/trs128_pytest.log
ST='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v*1000,1) for k,v in d["stages_ms"].items()})'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_r2.so paper_2312_15554_b200/build/lib_r2m6.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --workload transport --n 128 --steps 300 2>/dev/null | python -c "$ST") x3: $(python bench.py --workload transport --n 128 --tcells 3 --steps 100 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))')" >> gpurun_out/trs128.log
done; done
