B=paper_2312_15554_b200/build
for i in 1 2; do for lib in default $B/lib_tpk5.so $B/lib_tpk6.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  for args in "--n 128" "--n 128 --tcells 3"; do
  echo "$lib $args $(python bench.py --workload transport $args --steps 200 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})')" >> gpurun_out/r02bc_ab.log
  done
done; done
