mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cases --no-cpu > gpurun_out/torchrun1.log 2>&1; echo torchrun=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/torchrun_ref.log 2>&1; echo torchrun_ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --config C5 --gpus 1 --steps 5 --warmup 2 > gpurun_out/torchrun_c5.log 2>&1; echo torchrun_c5=$?
tail -c 700 gpurun_out/torchrun1.log; tail -c 300 gpurun_out/torchrun_c5.log
