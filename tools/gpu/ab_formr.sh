timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_runner.py -x -q -p no:cacheprovider > gpurun_out/r02am_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02am_pytest.log
for n in 200 256; do
  echo "n=$n" >> gpurun_out/r02am_ab.log
  POREFLOW_B200_PIPELINE=cufft bash tools/ab_libs.sh "--n $n --steps 100" paper_2312_15554_b200/build/lib_noformr.so default paper_2312_15554_b200/build/lib_noformr.so default >> gpurun_out/r02am_ab.log 2>&1
done
