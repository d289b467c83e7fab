import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_1904_04884_b200 import VolumeGeometry, ComplexField2D, SolverConfig, RegularizerWeights, fista
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
nx, ny, nz, iters = cfg[:4]
b = bench.make_hologram(cfg)
g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
for it in (10, 50, 100):
    vol, rep = fista(ComplexField2D(b, 10e-6, 632e-9), g, SolverConfig(weights=RegularizerWeights(cfg[6], cfg[7]), max_iters=it, tv_inner_iters=cfg[8]))
    rows_nz = sum(len(np.unique(p.rows)) for p in vol.planes)
    planes_nz = sum(1 for p in vol.planes if p.nnz)
    tiles = set()
    for k, p in enumerate(vol.planes):
        tiles.update(zip([k]*p.nnz, (p.rows // 64).tolist(), (p.cols // 64).tolist()))
    print(f"it {it}: nnz {vol.nnz} ({vol.nnz/(nx*ny*nz):.3%}) nonzero rows {rows_nz/(ny*nz):.1%} planes {planes_nz}/{nz} 64x64 tiles {len(tiles)/(nz*(ny//64)*(nx//64)):.1%}", flush=True)
