#!/usr/bin/env bash
# Final single-GPU measurement set of round 2 (run under gpurun from the repo root):
# headline bench + reference arm, launch lists and ncu --set full captures
# of the kernels changed late in the round. Outputs in gpurun_out/ (copied to profiles/).
set -u
out=gpurun_out
mkdir -p "$out"
timeout 900 python bench.py --steps 20 --warmup 5 > "$out/bench_n1.json" 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > "$out/bench_ref_n1.json" 2>&1
for q in 4 8; do
  for r in 8 16 32 64 128; do
    timeout 600 python bench.py --config llama7b-layer --rank "$r" --qbits "$q" --hold-rank \
      --no-cpu-baseline --e2e-steps 1 --steps 10 --warmup 3 > "$out/c3_r${r}_q${q}.json" 2>&1
  done
done
timeout 900 python bench.py --config qwen107b-stage --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > "$out/c4_n1.json" 2>&1
timeout 900 python bench.py --config mini-opt --steps 20 --warmup 5 --no-cpu-baseline > "$out/c1_n1.json" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file "$out/launches_default.csv" python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline --no-held-rank --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file "$out/launches_held.csv" python bench.py --steps 2 --warmup 3 --hold-rank \
  --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
for r in 64 128; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$out/launches_c3_r$r.csv" python bench.py --config llama7b-layer --rank $r \
    --qbits 8 --hold-rank --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 3 > /dev/null 2>&1
done
C3="python bench.py --config llama7b-layer --rank 128 --qbits 8 --hold-rank --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_cholblk" -s 2 -c 1 \
  -o "$out/full_k_cholblk" -f $C3 > "$out/full_k_cholblk.log" 2>&1
H="python bench.py --steps 2 --warmup 3 --hold-rank --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_chol32" -s 4 -c 1 \
  -o "$out/full_k_chol32" -f $H > "$out/full_k_chol32.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base function \
  -k "k_o5" -s 3 -c 1 -o "$out/full_k_o5" -f $H > "$out/full_k_o5.log" 2>&1
