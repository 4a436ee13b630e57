# 64^3 / 128^3 single cell: bench stages + ncu launch list (kernel durations vs the iteration time)
SS='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,3), round(d["ms_per_step"]*1000,2), "us/it", {k: round(v["ms"]*1000,2) for k,v in d["stages"].items()})'
for n in 64 128; do
  echo "n=$n $(python bench.py --n $n --steps 2000 --no-cpu-baseline 2>/dev/null | python -c "$SS")" >> gpurun_out/small64.log
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small64_launches.csv python tools/prof_stokes.py --n 64 --warmup 20 --iters 10 > /dev/null 2>&1
