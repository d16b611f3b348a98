mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-f2 --no-cpu-baseline > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo "bench2=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --impl reference --steps 1 --warmup 0 > gpurun_out/s2_ref.json 2> gpurun_out/s2_ref.err; echo "ref2=$?"
grep -c "NCCL INFO" gpurun_out/s2_bench.err
