# SYMV switch sweep on C3 (k_symv_whole variants) and C5 (k_symv_ring2 variants)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "" "DDG_WHOLE_STAGE=1" "DDG_WHOLE_WARPS=30" "DDG_WHOLE_PF=1" "DDG_WHOLE_PF=3" "DDG_WHOLE_STAGE=1 DDG_WHOLE_PF=2" \
         "DDG_RING_WHOLE=2" "DDG_RING_WHOLE=257" "DDG_RING_WHOLE=0" "DDG_WHOLE_STAGE=1 DDG_WHOLE_WARPS=30"; do
  env $v timeout 300 python tools/symv_probe.py C3 3 2>&1 | tail -1
done
for v in "" "DDG_RING_PF=1" "DDG_RING_PF=2" "DDG_RING_NB=3" "DDG_RING_TILES=2" "DDG_RING_V2=0"; do
  env $v timeout 300 python tools/symv_probe.py C5 3 2>&1 | tail -1
done
