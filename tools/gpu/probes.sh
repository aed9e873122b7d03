# Development probes (instrumented builds, not the product library): per-phase SM cycles of the
# large-tau factorisation (k_bfactor_lp) and of the EXPLICIT group kernel (k_iterate), then a
# `--set full` capture of k_bfactor_lp on the c5 pipeline (product build).
#   usage: bash tools/gpu/probes.sh [bf|it|ncu]...   (default: all)
what="${*:-bf it ncu}"
for w in $what; do
  case $w in
    bf) RS_NVCC_EXTRA=-DRS_BF_PHASES python -m paper_2105_05565_b200._build --force > /dev/null || exit 1
        python tools/probe_bf_phases.py c5 148 2>&1 | tee gpurun_out/bf_phases.txt
        python tools/probe_bf_phases.py k1 148 2>&1 | tee -a gpurun_out/bf_phases.txt ;;
    it) RS_NVCC_EXTRA=-DRS_IT_PHASES python -m paper_2105_05565_b200._build --force > /dev/null || exit 1
        python tools/probe_it_phases.py c5 240 2>&1 | tee gpurun_out/it_phases.txt
        python tools/probe_it_phases.py c2 148 2>&1 | tee -a gpurun_out/it_phases.txt ;;
    ncu) python -m paper_2105_05565_b200._build --force > /dev/null || exit 1
        timeout 800 ncu --set full --clock-control none --import-source on -k regex:"k_bfactor_lp" -c 1 \
          -o gpurun_out/bf_full python tools/prof_step.py c5 explicit 150 > gpurun_out/ncu_bf.log 2>&1 ;;
  esac
done
