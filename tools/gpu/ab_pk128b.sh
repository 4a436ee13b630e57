B=paper_2312_15554_b200/build
bash tools/ab_libs.sh "--n 128 --steps 300" default $B/lib_pk128b4.so $B/lib_pk128b5.so $B/lib_pk128b4np.so default > gpurun_out/r02az_ab.log 2>&1
for lib in default $B/lib_pk128b4.so $B/lib_pk128b4np.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --workload ensemble --n 128 --cells 16 --steps 200 2>/dev/null | cut -c80-130)" >> gpurun_out/r02az_ab.log
done
