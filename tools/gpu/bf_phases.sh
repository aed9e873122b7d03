# per-phase cycle probe of k_bfactor_lp (instrumented build, not the product library)
RS_NVCC_EXTRA=-DRS_BF_PHASES python -m paper_2105_05565_b200._build --force > /dev/null || exit 1
python tools/probe_bf_phases.py c5 148 2>&1 | tee gpurun_out/bf_phases.txt
python tools/probe_bf_phases.py k1 148 2>&1 | tee -a gpurun_out/bf_phases.txt
