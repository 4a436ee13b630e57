timeout 900 python -m pytest tests/test_gpu_fused_transport.py -x -q -p no:cacheprovider -k 256_vs_oracle > gpurun_out/t256.log 2>&1; echo "exit $?" >> gpurun_out/t256.log
python bench.py --n 64 --steps 500 --no-cpu-baseline > gpurun_out/n64.log 2>&1; echo "exit $?" >> gpurun_out/n64.log
