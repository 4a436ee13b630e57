# finalize: one-pass reduction of both partial arrays (product) vs two passes (lib_prev), and 256 threads (lib_fin256)
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v["ms"]*1000,1) for k,v in d["stages"].items()})'
for i in 1 2; do for n in 64 128 256; do
for lib in default paper_2312_15554_b200/build/lib_prev.so paper_2312_15554_b200/build/lib_fin256.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  st=$((n == 256 ? 100 : 600))
  echo "n=$n $lib $(python bench.py --n $n --steps $st --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/fin.log
done; done; done
