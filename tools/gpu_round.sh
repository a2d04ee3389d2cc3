#!/bin/bash
# One GPU-box pass: parity suite, smoke, bench (both arms), ncu launch list + full captures.
# Usage (from the build container): gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 python tools/probe_step.py > $OUT/step_timeline.json 2>&1
[ -z "${SKIP_SWEEP:-}" ] && timeout 1200 python tools/sweep.py --quick > $OUT/sweep.jsonl 2> $OUT/sweep.err
if [ -z "${SKIP_NCU:-}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --profile --steps 20 --warmup 3 > $OUT/launches.log 2>&1
python tools/launch_summary.py $OUT/launches.csv > $OUT/launch_summary.txt 2>&1
for K in k_score_bounded k_select_attend k_append; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
      -o $OUT/prof_$K python bench.py --profile --steps 5 > $OUT/ncu_$K.log 2>&1
done
fi
echo done
