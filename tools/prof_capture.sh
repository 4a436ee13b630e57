# Round capture on the GPU box (run under gpurun, one GPU):
#   bash tools/prof_capture.sh TAG
# GPU test suite + smoke, the bench line, the ncu launch list of the bench
# command itself, and --set full captures of the fused Stokes and transport
# passes (steady-state iterations).  Summarise here with tools/ncu_summary.py.
T=${1:-r01f}
set -x
python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; tail -n 3 gpurun_out/${T}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -n 1 gpurun_out/${T}_smoke.log
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench_err.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_bench_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu0.log 2>&1
python tools/prof_stokes.py --warmup 12 --iters 3 > gpurun_out/${T}_p0.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/${T}_launches.csv python tools/prof_stokes.py --warmup 3 --iters 3 > gpurun_out/${T}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pk|k_maxis|k_rs|k_stokes_finalize" --launch-skip 60 --launch-count 6 -o gpurun_out/${T}_full python tools/prof_stokes.py --warmup 12 --iters 3 > gpurun_out/${T}_ncu2.log 2>&1
python tools/prof_transport.py --warmup 8 --iters 3 > gpurun_out/${T}_p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_t_launches.csv python tools/prof_transport.py --warmup 3 --iters 3 > gpurun_out/${T}_ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tpk|k_taxis|k_trs|k_transport_finalize|finalize" --launch-skip 25 --launch-count 5 -o gpurun_out/${T}_t_full python tools/prof_transport.py --warmup 8 --iters 3 > gpurun_out/${T}_ncu4.log 2>&1
tail -n 2 gpurun_out/${T}_ncu0.log gpurun_out/${T}_ncu2.log gpurun_out/${T}_ncu4.log
