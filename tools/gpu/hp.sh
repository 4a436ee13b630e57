python tools/first_call.py > gpurun_out/hp_pinned.log 2>&1
POREFLOW_B200_PINNED_OUT_GB=0 python tools/first_call.py > gpurun_out/hp_ring.log 2>&1
POREFLOW_B200_PINNED_OUT_GB=0 POREFLOW_B200_HUGEPAGES=0 python tools/first_call.py > gpurun_out/hp_ring_nohp.log 2>&1
