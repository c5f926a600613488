#!/bin/bash
# Round-2 closing pass: whole GPU suite, smoke, bench lines (c4 default with cpu_baseline, c2, c3,
# c5 slice config if any, x8, x10, m12), c3 launch list and one --set full capture of its kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02final}; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
for c in c2 c3 x8 x10 m12; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > $O/l3.log 2>&1
NCU_COUNT=1 NCU_SKIP=1 timeout 900 bash tools/ncu_remote.sh ${1:-r02final}/ncu_c3_midr 'k_midr' python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['roofline']['bound'], d['clocks'].get('sm_mhz'))" 2>&1; done
