# small-m group-kernel grid (c2 EXPLICIT) and the dense XS gather (k_dense_xs_warp) on c2 IMPLICIT /
# c5 GRAM with ncu DRAM bytes
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --seeds 1"
for g in 148 64 32; do RS_IT_GRID=$g $B --config c2 --mode explicit > gpurun_out/m_c2_g$g.json 2>/dev/null; done
$B --config c2 --mode explicit > gpurun_out/m_c2_auto.json 2>/dev/null
for f in g148 g64 g32 auto; do python -c "
import json;d=json.loads(open('gpurun_out/m_c2_$f.json').read().strip().splitlines()[-1])
print('c2 explicit $f', round(d['value']), d['time_to_tol_s'], {k: round(v*1e3,2) for k, v in d['kernel_ms_per_step'].items() if v})"; done | tee gpurun_out/misc.txt
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv"
timeout 900 ncu $M -k regex:"k_dense_xs" -c 4 --log-file gpurun_out/tr_xs_c2.csv python tools/prof_step.py c2 implicit 4 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_dense_xs" -c 4 --log-file gpurun_out/tr_xs_c5.csv python tools/prof_step.py c5 gram 4 > /dev/null 2>&1
ls -la gpurun_out/tr_xs_c*.csv
