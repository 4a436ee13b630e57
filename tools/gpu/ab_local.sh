B=paper_2312_15554_b200/build
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q -p no:cacheprovider > gpurun_out/r02aj_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02aj_pytest.log
for n in 200 256; do
  echo "n=$n" >> gpurun_out/r02aj_ab.log
  POREFLOW_B200_PIPELINE=cufft bash tools/ab_libs.sh "--n $n --steps 60" $B/lib_locold.so default $B/lib_loc3.so $B/lib_loc1b4.so >> gpurun_out/r02aj_ab.log 2>&1
done
