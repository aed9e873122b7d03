set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/torchrun1_ref.json 2> gpurun_out/torchrun1_ref.err; echo rc=$?
timeout 600 python bench.py --config c1 --steps 50 --warmup 3 > gpurun_out/bench_c1.json 2>/dev/null; echo rc=$?
