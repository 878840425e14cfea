"""Debug: one small fused + split run (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import workloads as W
from tests import gpu_helpers as H
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 5
b = W.random_batch(seed, n=16, max_len=900, hq=8, hkv=2, d=128, decode_frac=0.5)
t = W.make_tensors(b, device="cuda")
for fused in (True, False):
    H.run_batch(b, t, C=512, decode_chunk=256, fused=fused)
torch.cuda.synchronize()
print("ok")
