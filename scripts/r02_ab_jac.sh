timeout 500 python -m pytest tests/test_gpu_large.py tests/test_gpu_shard.py -q -p no:cacheprovider --timeout 300 > gpurun_out/pt_jac.log 2>&1; tail -1 gpurun_out/pt_jac.log
for v in base nostream; do
  if [ $v = base ]; then lib=paper_2602_20226_b200/lib/libqtt.so; else lib=paper_2602_20226_b200/lib/libqtt_$v.so; fi
  for W in cfg4 cfg3; do
    QTT_LIB=$lib timeout 300 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v_$W.json 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v_$W.json').read().strip().splitlines()[-1]); print('$v $W', d['value'], d['ms_per_step'], d['jacobi']['sweeps_mean'])"
  done
done
QTT_COOP_WB=4 timeout 300 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_wb4.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ab_wb4.json').read().strip().splitlines()[-1]); print('base WB=4 cfg4', d['value'], d['ms_per_step'])"
