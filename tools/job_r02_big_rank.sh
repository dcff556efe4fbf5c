python -m pytest tests -m gpu -q --tb=short -k "larger_shapes or tensor_core_sweeps or compress_against or zero_tensors or effective_rank or engine" 2>&1 | tail -15 > gpurun_out/t_big.log
for r in 64 128; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3b_r$r.csv python bench.py --config llama7b-layer --rank $r --qbits 8 --hold-rank --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 3 > /dev/null 2>&1
done
for q in 4 8; do for r in 8 16 32 64 128; do
  timeout 600 python bench.py --config llama7b-layer --rank $r --qbits $q --hold-rank --no-cpu-baseline --e2e-steps 1 --steps 10 --warmup 3 > gpurun_out/c3c_r${r}_q${q}.json 2>&1
done; done
for r in 32 16 8 4; do RANK_R=$r DS=8 timeout 600 python tools/k5_scaling.py > gpurun_out/k5s_d8_r$r.log 2>&1; done
DS=8 timeout 600 python tools/d8_overlap.py > gpurun_out/d8_overlap.log 2>&1
