"""Line-granular DRAM model of the masked porous sweep (k_seg) on the dense
layout at the c4 bench geometry: bytes read at 32-B sector and 128-B line
granularity (ncu measures 30.9 GB per step; profiles/r02b_summary.md).

    python tools/c4_line_model_dense.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09242_b200 as dlb
L=600
cfg = dlb.CaseConfig(kind="porous", L=L, Ma=0.01, collision=dlb.LinkType.TRT, q=19, tau=1.0, upstream=40, downstream=40)
vox, phi = dlb.sphere_pack((L, L, L), radius=8.0, porosity=0.20, seed=20250611)
setup = dlb.init_porous(cfg, solid=(vox == 255))
idx = np.asarray(setup.chain_index); nz,ny,nx = idx.shape
G=4; nsx=(nx+G-1)//G
nd = np.pad(idx==2, ((0,0),(0,0),(0,nsx*G-nx)), constant_values=True)
listed = ~nd.reshape(nz,ny,nsx,G).all(-1)
pitch = ((nx+2+15)//16)*16; plane = pitch*(ny+2)
D=[(0,0,0),(-1,0,0),(1,0,0),(0,-1,0),(0,1,0),(0,0,-1),(0,0,1),(-1,-1,0),(1,1,0),(-1,1,0),(1,-1,0),(-1,0,-1),(1,0,1),(-1,0,1),(1,0,-1),(0,-1,-1),(0,1,1),(0,-1,1),(0,1,-1)]
z,y,s = np.nonzero(listed)
nl=len(z)
tot32=tot128=0
for cx,cy,cz in D:
    Y=(y-cy)%ny; Z=(z-cz)%nz
    base = (Z.astype(np.int64)*plane + Y.astype(np.int64)*pitch + 16 + s.astype(np.int64)*4 - cx)  # +16: x=0 at 16-elem aligned offset approx
    cells = (base[:,None] + np.arange(4)[None,:]).reshape(-1)
    tot32 += len(np.unique(cells//4)); tot128 += len(np.unique(cells//16))
print("dense layout: read GB at 32B %.2f at 128B %.2f" % (tot32*32/1e9, tot128*128/1e9))
