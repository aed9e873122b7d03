# per-iteration completion times of a c5 solve (development probe), then the normal build's lines
RS_NVCC_EXTRA=-DRS_IT_TIMES python -m paper_2105_05565_b200._build --force > /dev/null 2>&1 || exit 1
timeout 600 python tools/probe_it_times.py c5 600 > gpurun_out/it_times_c5.txt 2>&1
python -m paper_2105_05565_b200._build --force > /dev/null 2>&1
PYK="${PYK:-tau1024 or overlapped}" bash tools/gpu/check.sh
