timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k transport > gpurun_out/r02ak_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02ak_pytest.log
for i in 1 2; do for lib in paper_2312_15554_b200/build/lib_told.so default; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  for n in 200 256; do
  echo "$lib n=$n $(POREFLOW_B200_PIPELINE=cufft python bench.py --workload transport --n $n --steps 60 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), d["pipeline"], {k: round(v,4) for k,v in d["stages_ms"].items()})')" >> gpurun_out/r02ak_ab.log
  done
done; done
