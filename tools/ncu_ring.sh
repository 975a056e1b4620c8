# full ncu capture of one colour-sweep k_symv_ring launch per config (launch 5: a mid-sweep colour)
for c in ${CONFIGS:-C5 C3}; do
  timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring --launch-skip 5 -c 1 -o gpurun_out/ring_$c -f python tools/prof_solve.py $c > gpurun_out/ncu_ring_$c.log 2>&1
  echo "$c rc=$?"
done
