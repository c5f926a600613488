#!/bin/bash
# Round-2 final tree: whole GPU suite, smoke, the default bench line (c4, with cpu_baseline) and c3
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02close; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
for f in $O/bench_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], round(d['roofline']['frac'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
