# A/B helper for the append kernel: parity subset, bench lines, phase probe (tuning aid)
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests -m gpu -x -q -k "append or stats or extend or decode" > gpurun_out/ab/pytest.log 2>&1; echo "exit $?" >> gpurun_out/ab/pytest.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab/bench_$i.json 2>gpurun_out/ab/bench.err
done
timeout 300 python tools/probe_append.py > gpurun_out/ab/append.txt 2>&1
