# 2-GPU runs of the fused apply -> peer-store gather (bench.py --gather peer) against NCCL gathers
set -x
timeout 900 python -m pytest tests/test_peer_gather_gpu.py -m gpu -x -q > gpurun_out/peer_tests.log 2>&1; echo rc=$? >> gpurun_out/peer_tests.log
for c in ${CONFIGS:-small medium large}; do for g in ${GATHERS:-nccl nccl-root peer}; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29650 bench.py --gpus 2 --config $c --gather $g --no-stages --no-e2e > gpurun_out/pg_${c}_${g}.json 2> gpurun_out/pg_${c}_${g}.err
done; done
