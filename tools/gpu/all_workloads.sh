# every bench workload once (catches breakage outside the headline path): bash tools/gpu/all_workloads.sh TAG
T=${1:-all}
L=gpurun_out/${T}_workloads.log
run() { echo "== $*" >> $L; timeout 600 python bench.py "$@" 2>&1 | tail -2 | cut -c1-600 >> $L; }
run
run --impl reference --steps 2 --warmup 1 --cpu-budget 5
run --steps 300 --no-cpu-baseline
run --workload transport --steps 100
run --workload transport --n 128 --steps 200
run --workload transport --n 128 --tcells 3 --steps 100
run --workload ensemble --n 128 --steps 100
run --workload ensemble --n 64 --cells 8 --steps 200
run --workload ensemble --n 256 --cells 2 --steps 30
run --workload slab --n 128 --steps 30
run --workload slab --n 128 --steps 30 --slab-cufft
run --workload pipeline --n 128
run --workload pipeline --n 256 --geometry packing --stokes-only
run --n 64 --steps 1000 --no-cpu-baseline
run --n 128 --steps 400 --no-cpu-baseline
run --n 512 --steps 20 --no-cpu-baseline
run --n 200 --steps 30 --no-cpu-baseline
python tools/slab_rank_probe.py 1024 8 >> $L 2>&1 || echo "slab probe failed" >> $L
