"""One pinned text -> CSR ingest of config-2 edges (for ncu launch lists)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_09284_b200 as fb
from ingest_probe_lib import config2_text
text = config2_text()
pinned = torch.empty(len(text), dtype=torch.uint8, pin_memory=True); pinned.numpy()[:] = text
for _ in range(int(os.environ.get("REPS", "2"))):
    d = fb.DeviceGraph.from_edge_list(pinned.numpy()); d.close()
torch.cuda.synchronize()
print("ok")
