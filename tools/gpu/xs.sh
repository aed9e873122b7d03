# row-staged XS gather: IMPLICIT / GRAM parity subset, ncu DRAM bytes of the XS kernels on c2
# IMPLICIT and c5 GRAM, and the c2 IMPLICIT bench line
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "${PYK:-implicit or gram or tau1024 or xs or dual}" 2>&1 | tail -2 | tee gpurun_out/xs_pytest.log
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $M -k regex:"k_dense_xs" -c 4 --log-file gpurun_out/tr_xs_c2.csv python tools/prof_step.py c2 implicit 4 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_dense_xs" -c 4 --log-file gpurun_out/tr_xs_c5.csv python tools/prof_step.py c5 gram 4 > /dev/null 2>&1
timeout 600 python bench.py --config c2 --mode implicit --no-alt --no-e2e --no-cpu-baseline --seeds 1 --steps 50 > gpurun_out/xs_c2_implicit.json 2>/dev/null
python tools/showbench.py gpurun_out/xs_c2_implicit.json > gpurun_out/xs.txt 2>&1
