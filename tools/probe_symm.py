import os, socket, torch, torch.distributed as dist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import torch.distributed._symmetric_memory as symm
print([n for n in dir(symm) if not n.startswith("__")][:60])
t = symm.empty(1 << 20, dtype=torch.float32, device="cuda:0")
h = symm.rendezvous(t, dist.group.WORLD)
print("handle", type(h), [n for n in dir(h) if not n.startswith("_")])
for a in ("multicast_ptr", "buffer_ptrs", "signal_pad_ptrs", "world_size", "rank"):
    try: print(a, getattr(h, a))
    except Exception as e: print(a, "ERR", e)
print("has_multicast_support", getattr(symm, "has_multicast_support", lambda *a: "n/a")(torch.device("cuda:0").type, 0) if hasattr(symm, "has_multicast_support") else "n/a")
dist.destroy_process_group()
