set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_err.log
python tools/prof_stokes.py --warmup 12 --iters 3 > gpurun_out/p0.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r01e_launches.csv python tools/prof_stokes.py --warmup 3 --iters 3 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pk|k_maxis|k_rs|k_stokes_finalize" --launch-skip 60 --launch-count 6 -o gpurun_out/r01e_full python tools/prof_stokes.py --warmup 12 --iters 3 > gpurun_out/ncu2.log 2>&1
python tools/prof_transport.py --warmup 8 --iters 3 > gpurun_out/p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01e_t_launches.csv python tools/prof_transport.py --warmup 3 --iters 3 > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tpk|k_taxis|k_trs|k_transport_finalize|finalize" --launch-skip 25 --launch-count 5 -o gpurun_out/r01e_t_full python tools/prof_transport.py --warmup 8 --iters 3 > gpurun_out/ncu4.log 2>&1
tail -n 2 gpurun_out/ncu2.log gpurun_out/ncu4.log gpurun_out/p1.log
