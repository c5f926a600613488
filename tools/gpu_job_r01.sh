python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/suite3.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/suite3.txt 2>&1
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2>/dev/null
python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
cat gpurun_out/suite3.txt
