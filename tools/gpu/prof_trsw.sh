# ncu --set full of one RS_T launch, register-resident (k_trs_w) and k_trs, 256^3
for tw in 1 0; do
POREFLOW_B200_TRS_W=$tw ncu --set full --clock-control none --import-source on -k regex:"k_trs" --launch-skip 8 --launch-count 1 -o gpurun_out/trsw_$tw python tools/prof_transport.py --warmup 8 --iters 3 > gpurun_out/trsw_ncu_$tw.log 2>&1
done
