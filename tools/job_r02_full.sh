# ncu --set full captures (one launch each) of the kernels changed in round 2, after the same
# command ran clean without ncu; plus the GPU suite on the final code.
python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -12 > gpurun_out/t_all8.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-held-rank --e2e-steps 1 > gpurun_out/b8_pre.json 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-held-rank --e2e-steps 1"
for k in k_quant_pack k_cold_init k_chol32 k_o5; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 6 -c 1 \
    -o gpurun_out/r02_full_$k -f $B > gpurun_out/r02_full_$k.log 2>&1
done
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_gram_dmma_big|k_chol128" -s 4 -c 2 \
  -o gpurun_out/r02_full_c3r64 -f python bench.py --config llama7b-layer --rank 64 --qbits 8 --hold-rank \
  --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 3 > gpurun_out/r02_full_c3r64.log 2>&1
