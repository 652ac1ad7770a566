import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2502_17421_b200 import hta
from workloads.generators import config_workload
from workloads import fp8_cache
dev = torch.device("cuda:0")
w = config_workload("longchat7b_16k", seed=0)
x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
k8, ks = fp8_cache(w.k_cache); v8, vs = fp8_cache(w.v_cache)
k8, v8, ks, vs = k8.to(dev), v8.to(dev), ks.to(dev), vs.to(dev)
for _ in range(4):
    hta.hta_forward_fp8kv(x[0], k8, v8, ks, vs, x[3], x[4], mask)
torch.cuda.synchronize()
