# round-1 final validation (GPU box): tests, smoke, benches of every profiled config
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/final_suite.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" >> gpurun_out/final_suite.txt 2>&1
python bench.py > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2>/dev/null
python bench.py --config m12 --steps 3 --warmup 3 > gpurun_out/final_m12.json 2>/dev/null
python bench.py --config x8 --steps 5 --warmup 3 > gpurun_out/final_x8.json 2>/dev/null
python bench.py --config c2 --no-cpu-baseline > gpurun_out/final_c2.json 2>/dev/null
cat gpurun_out/final_suite.txt
