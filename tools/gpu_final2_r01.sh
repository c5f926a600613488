# round-1 closing validation (GPU box): tests, smoke, benches of every profiled config, then one
# ncu --set full capture of the dominant kernel of c4 / m12 / x8 (dram bytes -> roofline.traffic)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/f2_suite.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" >> gpurun_out/f2_suite.txt 2>&1
python bench.py > gpurun_out/f2_c4.json 2> gpurun_out/f2_c4.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f2_ref.json 2>/dev/null
python bench.py --config m12 --steps 3 --warmup 3 > gpurun_out/f2_m12.json 2>/dev/null
python bench.py --config x8 --steps 5 --warmup 3 > gpurun_out/f2_x8.json 2>/dev/null
python bench.py --config c2 --no-cpu-baseline > gpurun_out/f2_c2.json 2>/dev/null
python bench.py --config c3 --no-cpu-baseline > gpurun_out/f2_c3.json 2>/dev/null
bash tools/ncu_remote.sh f2_ncu_c4 k_passA python bench.py --steps 1 --warmup 3 --no-cpu-baseline
bash tools/ncu_remote.sh f2_ncu_m12 k_mana_rowS python bench.py --config m12 --steps 1 --warmup 3 --no-cpu-baseline
bash tools/ncu_remote.sh f2_ncu_x8 k_legs python bench.py --config x8 --steps 1 --warmup 3 --no-cpu-baseline
cat gpurun_out/f2_suite.txt
