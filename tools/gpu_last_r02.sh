#!/bin/bash
# Last round-2 GPU call: whole suite + smoke on the final tree, c3 --set full capture at its new grid
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02last; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
NCU_COUNT=1 NCU_SKIP=1 timeout 900 bash tools/ncu_remote.sh r02last/ncu_c3_midr 'k_midr' python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
tail -1 $O/smoke.log
