# factor phase probe (k_bfactor_lp SM cycles per phase) at nb = 1, 2 on c5 and k1
RS_NVCC_EXTRA=-DRS_BF_PHASES python -m paper_2105_05565_b200._build --force > /dev/null 2>&1 || exit 1
for nb in ${NBS:-1 2}; do
  RS_SB_NB=$nb RS_OV_SMS=0 timeout 300 python tools/probe_bf_phases.py c5 148 2>&1 | tail -12 > gpurun_out/bfp_c5_$nb.txt
done
python -m paper_2105_05565_b200._build --force > /dev/null 2>&1
