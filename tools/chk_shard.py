import sys, torch
sys.path.insert(0, "/root/repo")
import bench, paper_2211_07572_b200 as S
from paper_2211_07572_b200 import distributed as D
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec, kappa = bench.problem(cfg)
kind, n1, n2, b, ppw, desc = bench.CONFIGS[cfg]
sysm = S.assemble_fd5(spec)
dev = torch.device("cuda", 0)
rp, ci, v = (torch.from_numpy(a).to(dev) for a in (sysm.row_ptr, sysm.col_idx, sysm.values))
c = S.SolverConfig(b=b, compression=S.CompressionChoice.dense)
for trial in range(2):
    try:
        shards = [D.Shard(n1, n2, rp, ci, v, c, r, G) for r in range(G)]
        D.factorize_logical(shards)
        print("ok", [round(s.refresh_stats().t_stage1, 3) for s in shards], flush=True)
        for s in shards: s.close()
    except Exception as e:
        print("FAIL", e, flush=True)
import torch.distributed as dist
import os
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29544", RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl", device_id=dev)
try:
    sh = D.Shard(n1, n2, rp, ci, v, c, 0, 1)
    print("after nccl ok", flush=True)
except Exception as e:
    print("after nccl FAIL", e, flush=True)
dist.destroy_process_group()
