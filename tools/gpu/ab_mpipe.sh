POREFLOW_B200_M_PIPE=0 python tools/pk_variant_check.py /tmp/ref.npz > gpurun_out/r02n_chk.log 2>&1
POREFLOW_B200_M_PIPE=1 python tools/pk_variant_check.py /tmp/v.npz /tmp/ref.npz >> gpurun_out/r02n_chk.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_baseline_configs.py -x -q -p no:cacheprovider > gpurun_out/r02n_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02n_pytest.log
for mp in 0 1; do for n in 256 128; do echo "mpipe=$mp n=$n" >> gpurun_out/r02n_ab.log; POREFLOW_B200_M_PIPE=$mp bash tools/ab_libs.sh "--n $n --steps 200" default >> gpurun_out/r02n_ab.log 2>&1; done
POREFLOW_B200_M_PIPE=$mp python bench.py --workload ensemble --n 128 --cells 8 --steps 200 >> gpurun_out/r02n_ab.log 2>&1; done
