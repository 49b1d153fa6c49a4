#!/bin/bash
# StepSync (per-head select -> attend hand-off): the config B step with and
# without it, and with the selection padded to fewer CTAs per SM
mkdir -p gpurun_out
run() {
  timeout -k 10 300 python bench.py --steps 50 --warmup 10 --e2e-steps 20 --no-cpu --no-extra --max-iters 8 > gpurun_out/sync_$1.json 2>gpurun_out/sync_$1.err
  python - "$1" <<'PY'
import json,sys
v=sys.argv[1]
for l in open(f"gpurun_out/sync_{v}.json"):
    if l.startswith("{"):
        d=json.loads(l); print(v, "ms/step", d.get("ms_per_step"), "value", d.get("value"), "e2e", (d.get("e2e") or {}).get("value"))
PY
}
for r in 1 2; do
  unset CKV_SESSION_NO_STEPSYNC CKV_SEL_SMEM_KB
  run sync
  CKV_SESSION_NO_STEPSYNC=1 run nosync
  CKV_SEL_SMEM_KB=120 run pad120
  CKV_SEL_SMEM_KB=150 run pad150
done
