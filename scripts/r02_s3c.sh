O=gpurun_out/s3c; mkdir -p $O; rm -f gpurun_out/ab.txt
bash scripts/ab.sh base nopart base > /dev/null 2>&1; cp gpurun_out/ab.txt $O/ab.txt
grep -h -o '"jacobi": {[^}]*}' gpurun_out/ab_base.log gpurun_out/ab_nopart.log > $O/jac.txt
