# round-2 (session 3) evidence: --set full of one cfg4 encode step in the
# train step's form (level-major dout, FH_BWD_OVERWRITE), L2 flushed.
mkdir -p gpurun_out
export FH_OVERWRITE=1 FH_LM=1
timeout 300 python tools/time_encode.py cfg4 1 > gpurun_out/r02d_enc_cfg4_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none -k "regex:fwd_kernel|bwd_kernel|merge_shift" -s 32 -o gpurun_out/r02d_encode_cfg4lm -f python tools/time_encode.py cfg4 1 > gpurun_out/r02d_ncu_cfg4.log 2>&1
echo cfg4 rc=$?
for r in r02d_encode_cfg4lm; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
