import ctypes, os, torch, torch.distributed as dist
rank=int(os.environ["RANK"]); world=int(os.environ["WORLD_SIZE"]); torch.cuda.set_device(rank)
dist.init_process_group("gloo")
lib = ctypes.CDLL("libnccl.so.2")
uid = ctypes.create_string_buffer(128)
if rank == 0: print("getid", lib.ncclGetUniqueId(uid), flush=True)
obj=[uid.raw if rank==0 else None]; dist.broadcast_object_list(obj, src=0)
uid2 = ctypes.create_string_buffer(obj[0], 128)
class U(ctypes.Structure): _fields_=[("b", ctypes.c_char*128)]
u = U(); ctypes.memmove(ctypes.byref(u), uid2, 128)
comm = ctypes.c_void_p()
r = lib.ncclCommInitRank(ctypes.byref(comm), world, u, rank)
print("rank", rank, "init", r, flush=True)
