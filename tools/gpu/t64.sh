# 64^3 tile shapes: PK threads (96: 4 columns, one FFT round; 192: 8 columns, one round) and axis-1 threads (64: 8 columns)
V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v["ms"]*1000,1) for k,v in d["stages"].items()})'
for lib in default paper_2312_15554_b200/build/lib_pk64t96.so paper_2312_15554_b200/build/lib_pk64t192.so paper_2312_15554_b200/build/lib_m64t64.so paper_2312_15554_b200/build/lib_both.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib tests: $(timeout 600 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider -k 'oracle or cfg1' 2>&1 | tail -1)" >> gpurun_out/t64.log
  for i in 1 2; do
  echo "$lib $(python bench.py --n 64 --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "$V")" >> gpurun_out/t64.log
  done
  echo "$lib ens64 $(python bench.py --workload ensemble --n 64 --cells 8 --steps 200 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3))')" >> gpurun_out/t64.log
done
