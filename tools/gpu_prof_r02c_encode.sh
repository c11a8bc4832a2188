# round-2 final evidence: --set full of one encode
# step (cfg2 headline, cfg4 HBM regime), L2 flushed between steps.
mkdir -p gpurun_out
FH_OVERWRITE=1 timeout 300 python tools/time_encode.py cfg2 1 > gpurun_out/r02c_enc_cfg2_plain.log 2>&1 && \
FH_OVERWRITE=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|bwd_kernel|merge_shift" -o gpurun_out/r02c_encode_cfg2 -f python tools/time_encode.py cfg2 1 > gpurun_out/r02c_ncu_cfg2.log 2>&1
echo cfg2 rc=$?
FH_OVERWRITE=1 timeout 300 python tools/time_encode.py cfg4 1 > gpurun_out/r02c_enc_cfg4_plain.log 2>&1 && \
FH_OVERWRITE=1 timeout 1500 ncu --set full --clock-control none -k "regex:fwd_kernel|bwd_kernel|merge_shift" -s 30 -o gpurun_out/r02c_encode_cfg4 -f python tools/time_encode.py cfg4 1 > gpurun_out/r02c_ncu_cfg4.log 2>&1
echo cfg4 rc=$?
# summaries on the box (the reports themselves can exceed gpurun's 64 MiB copy-back)
for r in r02c_encode_cfg2 r02c_encode_cfg4; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
ls -la gpurun_out; du -sh gpurun_out
rm -f gpurun_out/r02c_encode_cfg4.ncu-rep
du -sh gpurun_out
