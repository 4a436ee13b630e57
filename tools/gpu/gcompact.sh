# cuFFT pipeline with solid-only multipliers: tests, then A/B at 200^3 (only path) and 256^3 forced
timeout 1200 python -m pytest tests/test_gpu_cufft_compact.py tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_steps.py -x -q -p no:cacheprovider > gpurun_out/gc_pytest.log 2>&1; echo "exit $?" >> gpurun_out/gc_pytest.log
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), d.get("pipeline"), {k: round(v["ms"],4) for k,v in d["stages"].items()})'
for i in 1 2; do for gc in 1 0; do
  echo "n=200 gc=$gc $(POREFLOW_B200_GCOMPACT=$gc python bench.py --n 200 --steps 100 --no-cpu-baseline 2>gpurun_out/gc_err.log | python -c "$SS")" >> gpurun_out/gc_ab.log
  echo "n=256 cufft gc=$gc $(POREFLOW_B200_PIPELINE=cufft POREFLOW_B200_GCOMPACT=$gc python bench.py --n 256 --steps 100 --no-cpu-baseline 2>>gpurun_out/gc_err.log | python -c "$SS")" >> gpurun_out/gc_ab.log
done; done
