# shared-memory carveout: driver default vs maximum (product), and the transport RS at 5 CTAs/SM
B=paper_2312_15554_b200/build
bash tools/ab_libs.sh "--steps 200" default $B/lib_carve_def.so default $B/lib_carve_def.so > gpurun_out/r02t_ab.log 2>&1
bash tools/ab_libs.sh "--n 128 --steps 300" default $B/lib_carve_def.so >> gpurun_out/r02t_ab.log 2>&1
for i in 1 2; do
for lib in default $B/lib_carve_def.so $B/lib_trs5.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --workload transport --steps 200 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})')" >> gpurun_out/r02t_ab.log
done; done
unset POREFLOW_B200_LIB
for lib in default $B/lib_carve_def.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --workload ensemble --n 128 --cells 8 --steps 200 2>/dev/null | cut -c1-140)" >> gpurun_out/r02t_ab.log
done
