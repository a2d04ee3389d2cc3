mkdir -p gpurun_out/s15
timeout 600 python -m pytest tests/test_gpu_bounded.py tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q > gpurun_out/s15/pytest.log 2>&1; echo "exit $?" >> gpurun_out/s15/pytest.log
for i in 1 2; do echo "$(timeout 300 python bench.py --no-cpu --no-dense --no-parity --steps 200 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')" >> gpurun_out/s15/cfg3.txt; done
timeout 300 python tools/probe_phases.py --clock > gpurun_out/s15/phases_clock.json 2>&1
timeout 300 python tools/probe_step.py > gpurun_out/s15/step.json 2>&1
