#!/bin/bash
# Full round pass: GPU tests, smoke, default bench (C2) + C4 + C3, launch list, ncu of the dominant kernel
# and of the C3 G-stage DGEMM.  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c4 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --nvtx --nvtx-include "csk_timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-acc --no-ne --no-ls --no-extra > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_share.py gpurun_out/launches_c2.csv 5 > gpurun_out/launch_share_c2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'cs_(bulk|tma|row)' -c 1 -o gpurun_out/prof_c2_main python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --no-ls --no-extra --cs-only > gpurun_out/ncu_main.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'gemm|Kernel2' -c 1 -o gpurun_out/prof_c3_gstage python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --no-extra > gpurun_out/ncu_gstage.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
for f in c2 c4 c3; do python -c "import json; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', round(d['value'],1), d['unit'], 'step', round(d['ms_per_step'],3), 'cs', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],3), 'ne', d['normal_equations'].get('ms'), d['normal_equations'].get('status'), 'speedup', d['speedup_vs_ne'], d['phases_ms'], d['accuracy'])" 2>&1 | tail -1; done
# NEXT items: rand_cholQR fused pass (C4) and the SRHT (k = 2n on C4's [A b])
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_pass_v3 -c 1 -o gpurun_out/prof_rc env REPS=1 python scripts/rc_once.py > gpurun_out/ncu_rc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srht_warp -c 1 -o gpurun_out/prof_srht env REPS=1 python scripts/srht_once.py > gpurun_out/ncu_srht.log 2>&1
timeout 300 python scripts/srht_once.py > gpurun_out/srht_c4.txt 2>&1; N=64 LOGD=24 timeout 300 python scripts/srht_once.py >> gpurun_out/srht_c4.txt 2>&1
timeout 300 python scripts/rc_once.py > gpurun_out/rc_c4.txt 2>&1; N=64 LOGD=24 timeout 300 python scripts/rc_once.py >> gpurun_out/rc_c4.txt 2>&1
cat gpurun_out/srht_c4.txt gpurun_out/rc_c4.txt
timeout 600 python bench.py --config srht > gpurun_out/bench_srht.json 2> gpurun_out/bench_srht.err
timeout 900 python bench.py --config rc --steps 10 > gpurun_out/bench_rc.json 2> gpurun_out/bench_rc.err
python -c "
import json
for f in ('srht','rc'):
    d=json.load(open('gpurun_out/bench_%s.json' % f)); r=d['roofline']; print(f, round(d['value'],1), d['unit'], 'step', round(d['ms_per_step'],3), 'kernel', round(r['kernel_ms'],3), 'frac', round(r['frac'],3))"
