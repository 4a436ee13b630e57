timeout 1200 python -m pytest tests/test_gpu_cufft_compact.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/gc2_pytest.log 2>&1; echo "exit $?" >> gpurun_out/gc2_pytest.log
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), d.get("pipeline"), {k: round(v["ms"],4) for k,v in d["stages"].items()})'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_gl_one.so paper_2312_15554_b200/build/lib_gl_two2.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib n=256 $(POREFLOW_B200_PIPELINE=cufft python bench.py --n 256 --steps 100 --no-cpu-baseline 2>>gpurun_out/gc_err.log | python -c "$SS")" >> gpurun_out/gc2_ab.log
done; done
