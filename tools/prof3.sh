# ncu launch lists of one three-level solve (C3 factor 4, C4 factor 2, C5 factor 4)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cf in "C3 4" "C4 2" "C5 4"; do set -- $cf
timeout 600 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/solve3_$1.csv python tools/prof_solve.py $1 3 $2 > gpurun_out/solve3_$1.log 2>&1; echo "$1 rc=$?"
done
