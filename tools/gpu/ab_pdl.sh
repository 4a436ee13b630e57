B=paper_2312_15554_b200/build
POREFLOW_B200_LIB=$B/lib_pdlearly.so python tools/pk_variant_check.py /tmp/v.npz > /dev/null 2>&1
python tools/pk_variant_check.py /tmp/ref.npz > gpurun_out/r02ay_chk.log 2>&1
POREFLOW_B200_LIB=$B/lib_pdlearly.so python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02ay_chk.log 2>&1
for n in 64 128 256; do
  echo "n=$n" >> gpurun_out/r02ay_ab.log
  bash tools/ab_libs.sh "--n $n --steps 300" default $B/lib_pdlearly.so default $B/lib_pdlearly.so >> gpurun_out/r02ay_ab.log 2>&1
done
for lib in default $B/lib_pdlearly.so; do
  if [ $lib = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  echo "$lib $(python bench.py --workload transport --n 64 --steps 300 2>/dev/null | cut -c60-120)" >> gpurun_out/r02ay_ab.log
  echo "$lib $(python bench.py --workload transport --n 128 --steps 300 2>/dev/null | cut -c60-120)" >> gpurun_out/r02ay_ab.log
done
