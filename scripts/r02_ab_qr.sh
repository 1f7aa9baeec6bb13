# A/B of the k_sweep QR trailing-update variants (cfg5 bench, no baselines)
rm -f gpurun_out/ab.txt
bash scripts/ab.sh base kc1 ld129 p16 base
cat gpurun_out/ab.txt
