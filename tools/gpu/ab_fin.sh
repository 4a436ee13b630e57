B=paper_2312_15554_b200/build
for n in 64 128 256; do
  echo "n=$n" >> gpurun_out/r02w_ab.log
  bash tools/ab_libs.sh "--n $n --steps 300" default $B/lib_fintriv.so $B/lib_norsf.so >> gpurun_out/r02w_ab.log 2>&1
done
