python tools/pk_variant_check.py /tmp/ref.npz > gpurun_out/r02ar_chk.log 2>&1
POREFLOW_B200_PK3=1 python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02ar_chk.log 2>&1
POREFLOW_B200_PK3=1 POREFLOW_B200_LIB=paper_2312_15554_b200/build/lib_pk3b2.so python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02ar_chk.log 2>&1
for i in 1 2; do
  echo "pk3=0" >> gpurun_out/r02ar_ab.log; POREFLOW_B200_PK3=0 bash tools/ab_libs.sh "--steps 300" default >> gpurun_out/r02ar_ab.log 2>&1
  echo "pk3=1" >> gpurun_out/r02ar_ab.log; POREFLOW_B200_PK3=1 bash tools/ab_libs.sh "--steps 300" default paper_2312_15554_b200/build/lib_pk3b2.so >> gpurun_out/r02ar_ab.log 2>&1
done
