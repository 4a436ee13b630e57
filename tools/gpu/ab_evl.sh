B=paper_2312_15554_b200/build
for n in 256 128; do
  echo "n=$n" >> gpurun_out/r02ac_ab.log
  bash tools/ab_libs.sh "--n $n --steps 300" default $B/lib_noevl.so default $B/lib_noevl.so >> gpurun_out/r02ac_ab.log 2>&1
done
