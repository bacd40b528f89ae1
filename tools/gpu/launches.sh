# ncu launch list of one bench step: tools/gpu/launches.sh CONFIG
c=${1:-C2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${c}_launches.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
python tools/gpu/summarize_launches.py gpurun_out/${c}_launches.csv
