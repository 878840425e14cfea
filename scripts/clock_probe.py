import sys, os, subprocess, time
sys.path.insert(0, os.getcwd())
import torch
from synth import workloads as W
from paper_2602_06072_b200 import packinfer as pk
b = W.cfg2_prefill(0)
t = W.make_tensors(b, device="cuda")
pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, b.hq // b.hkv, b.d, torch.bfloat16, "cuda")
out = torch.empty((b.total_q, b.hq, b.d), dtype=torch.bfloat16, device="cuda")
for _ in range(5): pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out)
torch.cuda.synchronize()
p = subprocess.Popen(["nvidia-smi","--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active","--format=csv,noheader","-lms","100"], stdout=subprocess.PIPE, text=True)
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(1000): pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out)
e1.record(); torch.cuda.synchronize(); p.terminate()
print("ms/step", e0.elapsed_time(e1)/1000)
print(p.stdout.read()[-1500:])
