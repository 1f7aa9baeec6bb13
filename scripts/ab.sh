# A/B benchmark of library variants: ab.sh name1 name2 ... ("base" = lib/libqtt.so)
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2602_20226_b200/lib/libqtt.so; else lib=paper_2602_20226_b200/lib/libqtt_$v.so; fi
  QTT_LIB=$lib timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.log 2>&1
  python -c "
import json,sys
l=json.loads([x for x in open('gpurun_out/ab_$v.log') if x.startswith('{')][0])
print('$v', l['value'], l['ms_per_step'], l['roofline']['prepass_ms_per_step'], l['roofline']['kernel_ms_per_step'], l['site_kernel_phase_share'])" >> gpurun_out/ab.txt 2>&1 || tail -3 gpurun_out/ab_$v.log >> gpurun_out/ab.txt
done
