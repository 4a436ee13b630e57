# transport RS_T tile-shape variants at 256^3 (correctness via the fused-transport tests, then timing)
B=paper_2312_15554_b200/build
for lib in $B/lib_trsr4.so $B/lib_trsr4b2.so; do
  POREFLOW_B200_LIB=$lib timeout 300 python -m pytest tests/test_gpu_fused_transport.py -x -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r02s_ab.log
done
for i in 1 2; do
for lib in default $B/lib_trsr4.so $B/lib_trsr4b2.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --workload transport --steps 200 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), {k: round(v,4) for k,v in d["stages_ms"].items()})')" >> gpurun_out/r02s_ab.log
done; done
