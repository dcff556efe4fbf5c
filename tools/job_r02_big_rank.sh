python -m pytest tests -m gpu -q --tb=short -k "larger_shapes or tensor_core_sweeps or compress_against or zero_tensors or outer_update" 2>&1 | tail -8 > gpurun_out/t_big2.log
for r in 64 128; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3d_r$r.csv python bench.py --config llama7b-layer --rank $r --qbits 8 --hold-rank --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 3 > /dev/null 2>&1
  timeout 600 python bench.py --config llama7b-layer --rank $r --qbits 8 --hold-rank --no-cpu-baseline --e2e-steps 1 --steps 10 --warmup 3 > gpurun_out/c3d_r${r}_q8.json 2>&1
done
for r in 4 8; do RANK_R=$r DS=8 timeout 600 python tools/k5_scaling.py > gpurun_out/k5s2_d8_r$r.log 2>&1; done
