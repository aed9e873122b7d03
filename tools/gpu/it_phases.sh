RS_NVCC_EXTRA=-DRS_IT_PHASES python -m paper_2105_05565_b200._build --force > /dev/null || exit 1
python tools/probe_it_phases.py c5 148 2>&1 | tee gpurun_out/it_phases.txt
python tools/probe_it_phases.py c2 148 2>&1 | tee -a gpurun_out/it_phases.txt
