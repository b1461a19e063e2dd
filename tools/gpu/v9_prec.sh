mkdir -p gpurun_out
for f in dit adjoint; do DBP_FFT=$f timeout 600 python tools/diag_fft_precision.py > gpurun_out/v9_prec_$f.jsonl 2> gpurun_out/v9_prec_$f.err; echo "$f rc=$?"; done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/v9b_gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/v9b_gputest.log
