# Round 2, call i: schedule / orthogonalisation choice by size (C2, C3, C5).
set -x
mkdir -p gpurun_out
for cfg in C2 C3 C5; do
  B="python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol"
  $B > gpurun_out/r02i_${cfg}_split_mgs.json 2>&1
  $B --schedule fused > gpurun_out/r02i_${cfg}_fused_mgs.json 2>&1
  $B --orth cgs2 > gpurun_out/r02i_${cfg}_split_cgs2.json 2>&1
  GSK_L2PF=0 $B > gpurun_out/r02i_${cfg}_split_mgs_pf0.json 2>&1
done
for f in gpurun_out/r02i_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres",
          round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
