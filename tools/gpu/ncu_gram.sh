# ncu evidence for the gram-mode (default) bench step on c2
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
CMD="python bench.py --mode ${MODE:-gram} --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --max-iter-tol 20"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${MODE:-gram}.csv $CMD > gpurun_out/ncu1.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_xpass_tma|k_gram_fused|k_bfactor_small|k_apply_ginv|k_update_vec}" -s ${SKIP:-20} -c ${COUNT:-5} -o gpurun_out/prof_${MODE:-gram} $CMD > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
