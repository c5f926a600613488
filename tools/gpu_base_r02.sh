#!/bin/bash
# Round-2 baseline: per-X-string rates of the round-1 kernels at N = 20..24 and one ncu --set full
# capture each of the N = 24 streamed pass A (k_passAs<24,12>) and its pass B (k_passBt<13,2>).
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/base_smi.txt
for spec in "20 524288 4096" "21 1048576 2048" "22 2097152 1024" "23 4194304 512" "24 8388608 256"; do
  python tools/rate.py $spec 3 >> gpurun_out/base_rates.txt 2>&1
done
cat gpurun_out/base_rates.txt
python tools/rate.py 24 8388608 16 1 > gpurun_out/base_plain24.log 2>&1 && \
NCU_COUNT=1 bash tools/ncu_remote.sh base_n24_passAs 'k_passAs' python tools/rate.py 24 8388608 16 1 && \
NCU_COUNT=1 bash tools/ncu_remote.sh base_n24_passBt 'k_passBt' python tools/rate.py 24 8388608 16 1
ls -la gpurun_out
