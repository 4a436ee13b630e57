POREFLOW_B200_RSFIX_TMA=0 python tools/pk_variant_check.py /tmp/ref.npz > gpurun_out/r02aa_chk.log 2>&1
python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02aa_chk.log 2>&1
POREFLOW_B200_M_PIPE=1 python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02aa_chk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_baseline_configs.py tests/test_gpu_parity.py tests/test_gpu_batch.py -x -q -p no:cacheprovider > gpurun_out/r02aa_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02aa_pytest.log
for n in 256 128; do
  for v in 0 1 0 1; do echo "n=$n rsfix_tma=$v" >> gpurun_out/r02aa_ab.log; POREFLOW_B200_RSFIX_TMA=$v bash tools/ab_libs.sh "--n $n --steps 300" default >> gpurun_out/r02aa_ab.log 2>&1; done
done
