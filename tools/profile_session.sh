#!/usr/bin/env bash
# One-GPU profiling session (run under gpurun from the repo root). Outputs land in
# gpurun_out/ (scratch); the summaries worth keeping are copied into profiles/ by hand.
#   bash tools/profile_session.sh [sanitize] [launches] [full] [sweep] [c4]
set -u
out=gpurun_out
mkdir -p "$out"
want() { [ $# -eq 0 ] && return 0; for a in "${ARGS[@]}"; do [ "$a" = "$1" ] && return 0; done; return 1; }
ARGS=("$@")
[ ${#ARGS[@]} -eq 0 ] && ARGS=(sanitize launches full sweep c4)

if want sanitize; then
  # memcheck / racecheck / synccheck of the smoke round (compress + fused outer update)
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool "$tool" --error-exitcode 9 \
      python -c "import __graft_entry__ as g; g.smoke()" > "$out/sanitize_$tool.log" 2>&1
    echo "sanitize $tool rc=$?" >> "$out/sanitize_summary.log"
  done
fi

if want launches; then
  # per-launch device times of one default bench run (controller applied) and of the
  # rank-held run: the kernels' shares of the round
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$out/launches_default.csv" python bench.py --steps 2 --warmup 3 \
    --no-cpu-baseline --no-held-rank --e2e-steps 1 > "$out/launches_default.log" 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$out/launches_held.csv" python bench.py --steps 2 --warmup 3 --hold-rank \
    --no-cpu-baseline --e2e-steps 1 > "$out/launches_held.log" 2>&1
fi

if want full; then
  # --set full of the changed kernels (one launch each, steady state)
  for k in k_quant_pack k_chol32 k_tc_sweep k_o5; do
    timeout 1200 ncu --set full --clock-control none --import-source on \
      -k "regex:$k" -s 40 -c 1 -o "$out/full_$k" -f python bench.py --steps 2 --warmup 3 \
      --hold-rank --no-cpu-baseline --e2e-steps 1 > "$out/full_$k.log" 2>&1
  done
fi

if want sweep; then
  # Llama-7B layer, rank sweep x int4 / int8 (rank held: the sweep is over r)
  for q in 4 8; do
    for r in 8 16 32 64 128; do
      timeout 600 python bench.py --config llama7b-layer --rank "$r" --qbits "$q" --hold-rank \
        --no-cpu-baseline --e2e-steps 1 --steps 10 --warmup 3 > "$out/c3_r${r}_q${q}.json" 2>&1
    done
  done
fi

if want c4; then
  timeout 900 python bench.py --config qwen107b-stage --steps 10 --warmup 3 --no-cpu-baseline \
    --e2e-steps 1 > "$out/c4_n1.json" 2>&1
  timeout 900 python bench.py --config mini-opt --steps 20 --warmup 5 --no-cpu-baseline \
    > "$out/c1_n1.json" 2>&1
fi
