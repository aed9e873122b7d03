set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bfactor_lp" -c 1 -o gpurun_out/prof_lp python tools/prof_step.py c5 explicit 150 > gpurun_out/ncu_lp.log 2>&1
RS_BF_RIGHT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bfactor_big" -c 1 -o gpurun_out/prof_rl python tools/prof_step.py c5 explicit 150 > gpurun_out/ncu_rl.log 2>&1
