#!/bin/bash
# Quick GPU iteration: parity suite + kernel launch list (device time per launch) + bench line.
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --profile --steps 20 --warmup 3 > $OUT/launches.log 2>&1
python tools/launch_summary.py $OUT/launches.csv > $OUT/launch_summary.txt 2>&1
if [ -z "${NO_BENCH:-}" ]; then
timeout 600 python bench.py --no-cpu ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
fi
