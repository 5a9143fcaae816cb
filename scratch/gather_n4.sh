# 1-GPU bench lines of the current build, then the gathers at N = 4
for c in small medium large; do CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in small large; do for g in nccl peer-all multimem; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 bench.py --gpus 4 --config $c --gather $g --no-stages --no-e2e > gpurun_out/pg4_${c}_${g}.json 2> gpurun_out/pg4_${c}_${g}.err
done; done
for f in gpurun_out/bench_*.json gpurun_out/pg4_*.json; do echo $f; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d[\"value\"], d[\"ms_per_step\"], d.get(\"gather_check\"), d.get(\"e2e\",{}).get(\"value\"))" $f; done
