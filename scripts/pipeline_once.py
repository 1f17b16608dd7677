"""One 4K RGB pipeline run (dd + ras+vi), for ncu captures of the
densification / dither / tonal kernels (scripts/ncu_geometry.sh)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_06747_b200 as sp
from oracle.oracle import synth
f = torch.from_numpy(synth(2160, 3840, 3, 0)).cuda()
mask, st, hist, _ = sp.run_pipeline(sp.Image(f), sp.PipelineConfig())
torch.cuda.synchronize()
print(mask.count, st.mse)
