#!/bin/bash
# Data-parallel DQN on 2 GPUs under NCCL protocol / algorithm settings (the gradient all-reduce
# is 1.35 MB per learn step, latency-bound): one bench line per setting.
for cfg in "" "NCCL_PROTO=LL128" "NCCL_PROTO=LL" "NCCL_ALGO=Tree" "NCCL_NVLS_ENABLE=0"; do
  env $cfg python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29521 bench.py --gpus 2 --no-configs --no-cpu-baseline > /tmp/nccl.jsonl 2>/dev/null
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("/tmp/nccl.jsonl").read().strip().splitlines()[-1])
s = d["secondary"]
print(sys.argv[1] or "default", {k: round(s[k]["value"] / 1e6, 2) for k in
      ("dqn_env_steps_per_s", "dqn_env_steps_per_s_precision3", "dqn_env_steps_per_s_pp_train", "dqn_env_steps_per_s_pp_infer")})
PY
done
