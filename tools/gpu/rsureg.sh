# Stokes RS at 256^3: u straight into registers (product) vs staged (lib_rsureg0)
timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_baseline_configs.py tests/test_gpu_slab.py -x -q -p no:cacheprovider > gpurun_out/rsureg_pytest.log 2>&1; echo "exit $?" >> gpurun_out/rsureg_pytest.log
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v["ms"],4) for k,v in d["stages"].items()})'
for i in 1 2 3; do for lib in default paper_2312_15554_b200/build/lib_rsureg0.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --steps 200 --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/rsureg_ab.log
done; done
