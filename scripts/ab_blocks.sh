# A/B of the cooperative Jacobi block count (QTT_COOP_BLOCKS) on one large workload
w=$1; shift
for nb in "$@"; do
  QTT_COOP_BLOCKS=$nb timeout 400 python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abb_$nb.log 2>&1
  python -c "
import json
l=json.loads([x for x in open('gpurun_out/abb_$nb.log') if x.startswith('{')][0])
print('$w', 'blocks=$nb', l['value'], l['ms_per_step'])" >> gpurun_out/ab.txt 2>&1 || tail -3 gpurun_out/abb_$nb.log >> gpurun_out/ab.txt
done
