set -x
nproc; lscpu | head -20; free -g; nvidia-smi; nvidia-smi topo -m
python - <<'PY'
import torch, time
print(torch.cuda.get_device_properties(0))
free,total=torch.cuda.mem_get_info(); print("mem", free/1e9, total/1e9)
for sz in [1<<20, 16<<20, 256<<20, 2<<30]:
    h=torch.empty(sz,dtype=torch.uint8).pin_memory(); d=torch.empty(sz,dtype=torch.uint8,device='cuda')
    for _ in range(3): d.copy_(h,non_blocking=True)
    torch.cuda.synchronize(); e0=torch.cuda.Event(True); e1=torch.cuda.Event(True)
    e0.record(); 
    for _ in range(5): d.copy_(h,non_blocking=True)
    e1.record(); torch.cuda.synchronize(); print("H2D",sz, 5*sz/e0.elapsed_time(e1)/1e6,"GB/s")
t=time.time(); h=torch.empty(30<<30,dtype=torch.uint8).pin_memory(); print("pin 30GB s", time.time()-t)
PY
