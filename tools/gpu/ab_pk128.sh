# PK variants at 128^3: single cell and the 8-cell ensemble
for pp in 0 1; do
  echo "pkpipe=$pp" >> gpurun_out/r02o_ab.log
  POREFLOW_B200_PK_PIPE=$pp bash tools/ab_libs.sh "--n 128 --steps 300" default >> gpurun_out/r02o_ab.log 2>&1
  POREFLOW_B200_PK_PIPE=$pp python bench.py --workload ensemble --n 128 --cells 8 --steps 200 2>/dev/null | cut -c1-200 >> gpurun_out/r02o_ab.log
done
for n in 64; do
  for mp in 0 1; do echo "n=$n mpipe=$mp" >> gpurun_out/r02o_ab.log; POREFLOW_B200_M_PIPE=$mp bash tools/ab_libs.sh "--n $n --steps 400" default >> gpurun_out/r02o_ab.log 2>&1; done
done
