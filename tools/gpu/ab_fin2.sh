B=paper_2312_15554_b200/build
for n in 256 128; do
  echo "n=$n" >> gpurun_out/r02ab_ab.log
  bash tools/ab_libs.sh "--n $n --steps 300" default $B/lib_nodb2.so $B/lib_nored.so $B/lib_fintriv2.so default >> gpurun_out/r02ab_ab.log 2>&1
  echo "grouped" >> gpurun_out/r02ab_ab.log
  POREFLOW_B200_GROUPED=1 bash tools/ab_libs.sh "--n $n --steps 300" default >> gpurun_out/r02ab_ab.log 2>&1
done
