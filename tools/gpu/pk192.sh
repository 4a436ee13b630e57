# PK with 192 threads (12 groups: one FFT round for the 12 sequences), 2 CTAs/SM, vs 128 threads (two rounds), 3 CTAs/SM
timeout 900 env POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_pk192.so python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider -k "oracle or headline" > gpurun_out/pk192_pytest.log 2>&1; echo "exit $?" >> gpurun_out/pk192_pytest.log
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v["ms"],4) for k,v in d["stages"].items()})'
for i in 1 2; do for lib in default paper_2312_15554_b200/build/lib_pk192.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib 256 $(python bench.py --steps 200 --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/pk192.log
  echo "$lib 128 $(python bench.py --n 128 --steps 400 --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/pk192.log
done; done
