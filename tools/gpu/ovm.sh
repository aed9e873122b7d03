# model-chosen SM split of the overlapped EXPLICIT pipeline: parity subset, then c5 / c4 / k1 with
# the model's split and c4 / k1 with forced splits (RS_OV_SMS)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "${PYK:-tau1024 or large_tau or overlapped or kernel_ridge or explicit or process_switches}" 2>&1 | tail -4 | tee gpurun_out/ovm_pytest.log
B="timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --seeds 1"
show() { python -c "
import json;d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$2', round(d['value']), round(d['time_to_tol_s']*1e3,2), d['roofline'].get('sms'), {k: round(v*1e3,2) for k, v in d['kernel_ms_per_step'].items() if v})" | tee -a gpurun_out/ovm.txt; }
$B > gpurun_out/ovm_c5.json 2>/dev/null; show gpurun_out/ovm_c5.json c5-model
$B --config c4 --max-iter-tol 20000 > gpurun_out/ovm_c4.json 2>/dev/null; show gpurun_out/ovm_c4.json c4-model
$B --config k1 --max-iter-tol 2000 > gpurun_out/ovm_k1.json 2>/dev/null; show gpurun_out/ovm_k1.json k1-model
for s in 80 96 120; do RS_OV_SMS=$s $B --config c4 --max-iter-tol 20000 > gpurun_out/ovm_c4_$s.json 2>/dev/null; show gpurun_out/ovm_c4_$s.json c4-$s; done
for s in 50 80 100; do RS_OV_SMS=$s $B --config k1 --max-iter-tol 2000 > gpurun_out/ovm_k1_$s.json 2>/dev/null; show gpurun_out/ovm_k1_$s.json k1-$s; done
