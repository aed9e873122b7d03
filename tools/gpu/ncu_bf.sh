python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 800 ncu --set full --clock-control none --import-source on -k regex:"k_bfactor_lp" -c 1 -o gpurun_out/bf_full python tools/prof_step.py c5 explicit 150 > gpurun_out/ncu_bf.log 2>&1
tail -2 gpurun_out/ncu_bf.log
