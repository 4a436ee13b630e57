# every bench workload once (catches breakage outside the headline path)
run() { echo "== $*" >> gpurun_out/r02av.log; timeout 600 python bench.py "$@" 2>&1 | tail -2 | cut -c1-400 >> gpurun_out/r02av.log; }
run --steps 30 --no-cpu-baseline
run --impl reference --steps 2 --warmup 1 --cpu-budget 5
run --workload transport --steps 50
run --workload transport --n 128 --tcells 3 --steps 50
run --workload ensemble --n 64 --cells 8 --steps 100
run --workload ensemble --n 256 --cells 2 --steps 30
run --workload slab --n 128 --steps 30
run --workload slab --n 128 --steps 30 --slab-cufft
run --workload pipeline --n 128
run --workload pipeline --n 256 --geometry packing --stokes-only
run --n 512 --steps 20 --no-cpu-baseline
run --n 200 --steps 30 --no-cpu-baseline
python tools/slab_rank_probe.py 1024 8 >> gpurun_out/r02av.log 2>&1 || echo "slab probe failed" >> gpurun_out/r02av.log
