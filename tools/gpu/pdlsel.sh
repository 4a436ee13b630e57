# early PDL trigger in the persistent / single-block passes (product) vs none (lib_nosel)
timeout 1500 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fused_transport.py tests/test_gpu_baseline_configs.py -x -q -p no:cacheprovider > gpurun_out/pdlsel_pytest.log 2>&1; echo "exit $?" >> gpurun_out/pdlsel_pytest.log
V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))'
for i in 1 2; do for lib in default nosel; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_$lib.so; fi
  echo "$lib 64: $(python bench.py --n 64 --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "$V") 128: $(python bench.py --n 128 --steps 400 --no-cpu-baseline 2>/dev/null | python -c "$V") 256: $(python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "$V") ens128: $(python bench.py --workload ensemble --n 128 --steps 100 2>/dev/null | python -c "$V") T64: $(python bench.py --workload transport --n 64 --steps 600 2>/dev/null | python -c "$V") T256: $(python bench.py --workload transport --n 256 --steps 100 2>/dev/null | python -c "$V")" >> gpurun_out/pdlsel.log
done; done
