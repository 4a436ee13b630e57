# finalize: done flag read with the partials (product) vs before them (lib_prev)
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fused_transport.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/fin2_pytest.log 2>&1; echo "exit $?" >> gpurun_out/fin2_pytest.log
V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_prev.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib 64: $(python bench.py --n 64 --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "$V") 128: $(python bench.py --n 128 --steps 400 --no-cpu-baseline 2>/dev/null | python -c "$V") T128: $(python bench.py --workload transport --n 128 --steps 300 2>/dev/null | python -c "$V") T64: $(python bench.py --workload transport --n 64 --steps 600 2>/dev/null | python -c "$V")" >> gpurun_out/fin2.log
done; done
