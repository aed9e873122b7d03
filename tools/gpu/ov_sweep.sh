# OV_SMS sweep of the overlapped EXPLICIT pipeline on the c5 line (development)
python -c "import __graft_entry__ as g; g.build()" || exit 1
for r in ${SWEEP:-18 22 26 30}; do
  sed -i "s/^constexpr int OV_SMS = [0-9]*;/constexpr int OV_SMS = $r;/" paper_2105_05565_b200/csrc/rs_internal.cuh
  python -m paper_2105_05565_b200._build > /dev/null 2>&1 || exit 1
  timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --seeds 2 > gpurun_out/ov_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ov_$r.json').read().strip().splitlines()[-1])
print('OV_SMS $r', round(d['value']), round(d['time_to_tol_s']*1e3,2), {k: round(v*1e3,2) for k, v in d['kernel_ms_per_step'].items() if v})" | tee -a gpurun_out/ov_sweep.txt
done
