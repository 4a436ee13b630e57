V='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],3), round(d["voxel_iters_per_s"]/1e9,2))'
for i in 1 2; do for lib in default f1024u4 r02e; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_$lib.so; fi
  echo "$lib cfg2: $(python bench.py --workload pipeline --n 128 2>/dev/null | python -c "$V") cfg3: $(python bench.py --workload pipeline --n 256 --geometry packing --stokes-only 2>/dev/null | python -c "$V")" >> gpurun_out/pipe_bisect.log
done; done
