"""4K RGB pipeline wall time (device, CUDA events) per ORAS kernel variant."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import _lib
from oracle.oracle import synth
lib = _lib.load()
f = torch.from_numpy(synth(2160, 3840, 3, 0)).cuda()
cfg = sp.PipelineConfig()
variants = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]] or [(6, 1, 0, 0), (6, 1, 0, 1)]
for v, tf, cp, gl in variants * 2:
    lib.sp_oras_variant(v)
    lib.sp_tile_fused(tf)
    lib.sp_channel_parallel(cp)
    lib.sp_graph_loop(gl)
    sp.solver._POOL.clear()
    sp.run_pipeline(sp.Image(f), cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        mask, st, hist, _ = sp.run_pipeline(sp.Image(f), cfg)
    e1.record()
    torch.cuda.synchronize()
    print(f"oras {v} tile_fused {tf} chan_par {cp} graph_loop {gl}: {e0.elapsed_time(e1) / 2:.1f} ms/pipeline  mse={st.mse:.9f} "
          f"dd_mse={hist[-1][2]:.9f} count={mask.count}", flush=True)
