# usage: CFG=c2 MODE=gram ITERS=8 KREGEX='k_a|k_b' COUNT=4 bash tools/gpu/ncu_step.sh
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
TAG=${TAG:-${CFG:-c2}_${MODE:-gram}}
CMD="python tools/prof_step.py ${CFG:-c2} ${MODE:-gram} ${ITERS:-8}"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu1_$TAG.log 2>&1
if [ -n "$KREGEX" ]; then
ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -c ${COUNT:-4} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu2_$TAG.log 2>&1
fi
cat gpurun_out/plain_$TAG.log; tail -n 3 gpurun_out/ncu1_$TAG.log gpurun_out/ncu2_$TAG.log
