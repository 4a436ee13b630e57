# per-iteration fixed costs at 64^3 / 128^3: finalize and RS-fix launches removed (timing only)
B=paper_2312_15554_b200/build
for n in 64 128; do
  echo "n=$n" >> gpurun_out/r02p_ab.log
  bash tools/ab_libs.sh "--n $n --steps 400" default $B/lib_norsf.so $B/lib_nofin.so $B/lib_noboth.so >> gpurun_out/r02p_ab.log 2>&1
done
