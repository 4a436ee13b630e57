# upper bounds of removing the RS-fix launch (NORSF) / the finalize's work (FINTRIV) at 64 / 128 / 256
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v["ms"]*1000,1) for k,v in d["stages"].items()})'
for n in 64 128 256; do
for lib in default paper_2312_15554_b200/build/lib_norsf.so paper_2312_15554_b200/build/lib_fintriv.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  st=$((n == 256 ? 100 : 600))
  echo "n=$n $lib $(python bench.py --n $n --steps $st --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/abl_small.log
done; done
