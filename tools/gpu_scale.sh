# Weak-scaling bench at N = 1, 2, 4 on one box (run with gpurun --gpus 4).
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/s_topo.txt 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/s_n1.json 2> gpurun_out/s_n1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/s_n$N.json 2> gpurun_out/s_n$N.err
done
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/s_multi.log 2>&1
