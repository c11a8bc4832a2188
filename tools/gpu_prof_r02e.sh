# round-2 final evidence (session 3): cfg4 encode step in the train form
# (level-major dout, overwrite, in-pass replicas) under --set full; the
# default bench and its launch list.
mkdir -p gpurun_out
export FH_OVERWRITE=1 FH_LM=1
timeout 300 python tools/time_encode.py cfg4 1 > gpurun_out/r02e_enc_cfg4_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none -k "regex:bwd_kernel|rep_reduce" -s 39 -c 13 -o gpurun_out/r02e_encode_cfg4lm -f python tools/time_encode.py cfg4 1 > gpurun_out/r02e_ncu_cfg4.log 2>&1
echo cfg4 rc=$?
python tools/ncu_summary.py gpurun_out/r02e_encode_cfg4lm.ncu-rep > gpurun_out/r02e_encode_cfg4lm_summary.txt 2>&1
ncu -i gpurun_out/r02e_encode_cfg4lm.ncu-rep --page raw --csv > gpurun_out/r02e_encode_cfg4lm_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
unset FH_OVERWRITE FH_LM
timeout 600 python bench.py > gpurun_out/r02e_bench.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02e_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_ncu_launch.log 2>&1
echo launches rc=$?
du -sh gpurun_out
