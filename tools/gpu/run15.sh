make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "csr" > gpurun_out/gpu_tests_csr.log 2>&1; echo "csr tests rc=$?"; tail -2 gpurun_out/gpu_tests_csr.log
for c in C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], 'ms', round(d['ms_per_step'],3), 'roof', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:10]})"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:csr_spmm_kernel -c 6 --csv --log-file gpurun_out/c5_spmm_l2.csv python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
grep -v "^==" gpurun_out/c5_spmm_l2.csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for row in r[1:]:
    d=dict(zip(h,row)); print(d['ID'], d['Metric Name'], d['Metric Value'])"
