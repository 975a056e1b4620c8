# k_symv_ring2 on C5: the epilogue's tail strip as a lane-column walk (default) vs row by row,
# and the probes (no strip, bare epilogue, copy-only consumers)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "" "DDG_RING2_ROWSTRIP=1" "" "DDG_RING2_ROWSTRIP=1" "DDG_RING2_BARE_EPI=2" "DDG_RING2_BARE_EPI=1" "DDG_RING2_COPYONLY=1 DDG_RING2_BARE_EPI=1"; do
  env $v timeout 300 python tools/symv_probe.py ${1:-C5} 3 2>&1 | tail -1
done
