"""One qgm_index_build (build_qgroup_index<u32>, the API's read-side index of
Alg. 1) over a bench config's first batch, after a warm-up build -- for ncu
(--profile-from-start off: only the second build is captured)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1403_1706_b200 as qgm  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
ref, cb = bench.make_reference(qgm, cfg)
codes, lengths = bench.make_block(qgm, cfg, ref, cb, 0)
ctx = qgm.Context(0)
reads = qgm.Reads.from_codes(ctx, codes, lengths, cfg["rlen"])
idx = qgm.Index.build(ctx, reads, cfg["q"])
del idx
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
idx = qgm.Index.build(ctx, reads, cfg["q"])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(idx.info)
