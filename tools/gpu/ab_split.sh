POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_nosplit.so python tools/pk_variant_check.py /tmp/ref.npz > gpurun_out/r02af_chk.log 2>&1
python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02af_chk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_baseline_configs.py -x -q -p no:cacheprovider > gpurun_out/r02af_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02af_pytest.log
for n in 256 128; do
  echo "n=$n" >> gpurun_out/r02af_ab.log
  bash tools/ab_libs.sh "--n $n --steps 300" default paper_2312_15554_b200/build/lib_nosplit.so default paper_2312_15554_b200/build/lib_nosplit.so >> gpurun_out/r02af_ab.log 2>&1
done
