# large-tau parity + c5 bench line (product build), then the factor phase probe (instrumented build)
bash tools/gpu/quick_c5.sh
bash tools/gpu/bf_phases.sh > /dev/null 2>&1
cat gpurun_out/bf_phases.txt
