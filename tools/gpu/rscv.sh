# compact RS occupancy: select-form merge (132 regs) and/or the maximum carveout (5 CTAs/SM by shared memory)
timeout 900 env POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_selcv.so python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider -k "oracle or headline" > gpurun_out/rscv_pytest.log 2>&1; echo "exit $?" >> gpurun_out/rscv_pytest.log
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v["ms"],4) for k,v in d["stages"].items()})'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_sel.so paper_2312_15554_b200/build/lib_cv.so paper_2312_15554_b200/build/lib_selcv.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --steps 200 --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/rscv.log
done; done
