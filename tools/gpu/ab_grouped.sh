POREFLOW_B200_GROUPED=0 python tools/pk_variant_check.py /tmp/ref.npz > gpurun_out/r02x_chk.log 2>&1
python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02x_chk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_baseline_configs.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r02x_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02x_pytest.log
for n in 64 128 256; do
  for gr in 0 1; do echo "n=$n grouped=$gr" >> gpurun_out/r02x_ab.log; POREFLOW_B200_GROUPED=$gr bash tools/ab_libs.sh "--n $n --steps 300" default >> gpurun_out/r02x_ab.log 2>&1; done
done
for gr in 0 1; do echo "grouped=$gr $(POREFLOW_B200_GROUPED=$gr python bench.py --workload ensemble --n 128 --cells 8 --steps 200 2>/dev/null | cut -c1-120)" >> gpurun_out/r02x_ab.log; done
