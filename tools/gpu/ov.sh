# quick: large-tau / explicit parity subset + c5 line + k_iterate phases (instrumented build)
bash tools/gpu/quick_c5.sh
RS_NVCC_EXTRA=-DRS_IT_PHASES python -m paper_2105_05565_b200._build --force > /dev/null 2>&1 || exit 1
python tools/probe_it_phases.py c5 264 2>&1 | tee gpurun_out/it_phases.txt
