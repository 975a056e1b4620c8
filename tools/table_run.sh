python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/table_sweep.py A > gpurun_out/table_A.txt 2> gpurun_out/table_A.err; echo "A rc=$?"
timeout 1500 python tools/table_sweep.py F > gpurun_out/table_F.txt 2> gpurun_out/table_F.err; echo "F rc=$?"
