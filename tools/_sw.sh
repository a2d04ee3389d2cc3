mkdir -p gpurun_out/s3
for cfg in "PT_NO_SPLIT=1 PT_SB_STATIC=1" "PT_NO_SPLIT=1 PT_SB_CHUNK=2" "PT_NO_SPLIT=1 PT_SB_CHUNK=4" "PT_NO_SPLIT=1 PT_SB_CHUNK=8" "PT_NO_SPLIT=0 PT_SB_STATIC=1" "PT_NO_SPLIT=0 PT_SB_CHUNK=4" "PT_NO_SPLIT=0 PT_SB_CHUNK=8"; do
  echo "$cfg $(env $cfg timeout 300 python bench.py --no-cpu --no-dense --no-parity --steps 100 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["achieved"])')" >> gpurun_out/s3/sweep.txt
done
