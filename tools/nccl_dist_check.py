"""bench.Dist over NCCL at world size 1 on one GPU: init with device_id and the
long timeout, barrier, max, object and tensor gathers (the calls the
multi-GPU bench makes; the box has one GPU, so more ranks run under gloo)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29561", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
d = bench.Dist(1, 0, use_cuda=True)
d.barrier()
print("backend", d.backend, "max", d.max(2.5), "objs", d.objects({"r": 0}),
      "frames", [f.shape for f in d.tensors(torch.ones((4, 6, 3), dtype=torch.uint8, device="cuda"))])
d.close()
print("nccl dist ok")
