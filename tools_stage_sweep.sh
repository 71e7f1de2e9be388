# staged launches vs the flow kernel: HPEZ_STAGE_MIN = smallest level (points) run staged
for sm in 9223372036854775807 100000000 10000000 1000000 100000; do
  echo "cfg4 STAGE_MIN=$sm $(HPEZ_STAGE_MIN=$sm python tools_cfg4.py --cfg 4 --no-oracle --iters 4 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["compress_ms"], d["decompress_ms"], d["num_launches"])')"
done
for sm in 9223372036854775807 30000000 3000000 300000; do
  echo "cfg2 STAGE_MIN=$sm $(HPEZ_STAGE_MIN=$sm python tools_sweep_time.py)"
done
