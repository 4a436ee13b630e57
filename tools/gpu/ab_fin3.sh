POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_fin1.so python tools/pk_variant_check.py /tmp/ref.npz > gpurun_out/r02ao_chk.log 2>&1
python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02ao_chk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_baseline_configs.py -x -q -p no:cacheprovider > gpurun_out/r02ao_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02ao_pytest.log
for n in 256 128; do
  echo "n=$n" >> gpurun_out/r02ao_ab.log
  bash tools/ab_libs.sh "--n $n --steps 300" paper_2312_15554_b200/build/lib_fin1.so default paper_2312_15554_b200/build/lib_fin1.so default >> gpurun_out/r02ao_ab.log 2>&1
done
