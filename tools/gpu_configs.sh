# bench.py config modes on one GPU: C3 (six tiles, loopback), C4 (768^2), and
# the N > 1 code paths as processes sharing the GPU (FV3B_SAME_GPU=1: no timing meaning)
set -x
summ() { python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(json.dumps({k: d.get(k) for k in ('value','ms_per_step','scaling','n_gpus')} | {'workload': d['config']['workload'], 'decomp': d['config']['decomposition'], 'halo': (d.get('method') or d['config']).get('halo'), 'e2e_ms': d['e2e']['ms_per_step']}))"; }
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu 2>&1 | summ
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu 2>&1 | summ
FV3B_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c4 --halo peer --steps 2 --warmup 3 2>&1 | summ
FV3B_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 6 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 6 --config c3 --halo peer --steps 2 --warmup 3 2>&1 | summ
# (the default NCCL halo path cannot run here: NCCL needs one GPU per rank and gloo cannot
#  move CUDA tensors; its packing is covered by the loopback 'packed' GPU tests)
