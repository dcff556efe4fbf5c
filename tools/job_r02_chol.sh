#!/usr/bin/env bash
# CholQR rework check: parity of every compress path, then C3 (Llama-7B layer) at r = 64 / 128
# with the blocked and the unblocked factorisation, the headline bench, and launch lists.
set -u
out=gpurun_out
mkdir -p "$out"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "compress or cold" > "$out/chol_tests.log" 2>&1
echo "tests rc=$?" >> "$out/chol_tests.log"
for r in 64 128; do
  for b in 1 0; do
    timeout 600 python bench.py --config llama7b-layer --rank "$r" --qbits 8 --hold-rank \
      --no-cpu-baseline --e2e-steps 1 --steps 10 --warmup 3 --option cholqr_blocked=$b \
      > "$out/c3_r${r}_b${b}.json" 2>&1
  done
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > "$out/bench_n1.json" 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --hold-rank > "$out/bench_n1_held.json" 2>&1
for r in 64 128; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$out/launches_c3_r${r}.csv" python bench.py --config llama7b-layer --rank "$r" \
    --qbits 8 --hold-rank --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 3 > /dev/null 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file "$out/launches_held.csv" python bench.py --steps 2 --warmup 3 --hold-rank \
  --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
