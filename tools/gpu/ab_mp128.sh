# persistent axis-1 pass variants at 128^3 (ring depth, CTAs per SM): single cell + 8-cell ensemble
B=paper_2312_15554_b200/build
bash tools/ab_libs.sh "--n 128 --steps 300" default $B/lib_mp3.so $B/lib_mpb4.so $B/lib_mp3b3.so > gpurun_out/r02r_ab.log 2>&1
for lib in default $B/lib_mp3.so $B/lib_mpb4.so $B/lib_mp3b3.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --workload ensemble --n 128 --cells 8 --steps 200 2>/dev/null | cut -c1-140)" >> gpurun_out/r02r_ab.log
done
