mkdir -p gpurun_out/s10
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/s10/pytest.log 2>&1; tail -4 gpurun_out/s10/pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 > gpurun_out/s10/bench_torchrun.json 2> gpurun_out/s10/bench_torchrun.err; head -c 600 gpurun_out/s10/bench_torchrun.json; echo; tail -3 gpurun_out/s10/bench_torchrun.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/s10/bench_ref_torchrun.json 2> gpurun_out/s10/bench_ref_torchrun.err; head -c 300 gpurun_out/s10/bench_ref_torchrun.json; echo
