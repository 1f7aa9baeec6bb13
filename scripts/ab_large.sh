# A/B of library variants on a large-path workload: ab_large.sh WORKLOAD name1 name2 ...
w=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2602_20226_b200/lib/libqtt.so; else lib=paper_2602_20226_b200/lib/libqtt_$v.so; fi
  QTT_LIB=$lib timeout 400 python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abl_$v.log 2>&1
  python -c "
import json
l=json.loads([x for x in open('gpurun_out/abl_$v.log') if x.startswith('{')][0])
print('$w', '$v', l['value'], l['ms_per_step'], l['jacobi_sweeps'])" >> gpurun_out/ab.txt 2>&1 || tail -3 gpurun_out/abl_$v.log >> gpurun_out/ab.txt
done
