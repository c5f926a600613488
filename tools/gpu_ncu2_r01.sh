# round-1: ncu --set full of the dominant staged kernel of c4 (k_passA10s) and of every leg of one x8 sweep
mkdir -p gpurun_out
NCU_COUNT=2 bash tools/ncu_remote.sh f3_ncu_c4 k_passA10s python bench.py --steps 1 --warmup 3 --no-cpu-baseline
NCU_COUNT=3 bash tools/ncu_remote.sh f3_ncu_x8 k_legs python bench.py --config x8 --steps 1 --warmup 3 --no-cpu-baseline
tail -2 gpurun_out/f3_ncu_c4.ncu.log gpurun_out/f3_ncu_x8.ncu.log
