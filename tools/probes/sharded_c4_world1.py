import os, sys, json, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import bench
print(json.dumps(bench.sharded_config4(0, 0, 1, dist)))
print(json.dumps(bench.comm_info()))
dist.destroy_process_group()
