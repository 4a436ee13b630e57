python tools/pk_variant_check.py /tmp/v.npz > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_batch.py tests/test_gpu_baseline_configs.py tests/test_gpu_parity.py tests/test_native_abi.py -x -q -p no:cacheprovider > gpurun_out/r02be_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02be_pytest.log
python tools/e2e_probe2.py > gpurun_out/r02be.log 2>&1
python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"]/1e9, d["e2e"])' >> gpurun_out/r02be.log
