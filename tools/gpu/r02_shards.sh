# cfg5 shards on one GPU (projection of the N-GPU run), then ncu of the 8-way shard
mkdir -p gpurun_out
python tools/shard_bench.py > gpurun_out/cfg5_shards.jsonl 2> gpurun_out/cfg5_shards.err; cat gpurun_out/cfg5_shards.jsonl
cat > /tmp/shard8.py <<'PY'
import math, sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1607_00291_b200 as tc
from paper_1607_00291_b200 import dist as tdist
import workloads as W
case = W.cfg5()
A, B, _ = W.make_tensors(case, "cuda")
rg = tdist.shard_ranges(8, 0, case.lens, "abc")
shape = tdist.shard_shape(case.lab_c, case.lens, rg)
Cs = W.colmajor_view(torch.empty(math.prod(shape), dtype=torch.float64, device="cuda"), shape)
for _ in range(2):
    tdist.contract_shard(case.spec, A, B, Cs, rg, 1.0, 0.0)
torch.cuda.synchronize()
PY
timeout 300 python /tmp/shard8.py && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tc_dmma -s 1 -c 1 -o gpurun_out/prof_shard8 python /tmp/shard8.py > gpurun_out/ncu_shard8.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_shard8.ncu-rep > gpurun_out/summary_shard8.txt 2>&1; head -20 gpurun_out/summary_shard8.txt; rm -f gpurun_out/prof_shard8.ncu-rep
