"""Traffic model of 128-B brick layouts for the c4 porous sweep (listed
bricks written whole, reads = bricks touched by the shifted listed set,
perfect L2 reuse assumed; profiles/r02b_summary.md).

    python tools/c4_brick_model.py
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
nd = idx==2
D=[(0,0,0),(-1,0,0),(1,0,0),(0,-1,0),(0,1,0),(0,0,-1),(0,0,1),(-1,-1,0),(1,1,0),(-1,1,0),(1,-1,0),(-1,0,-1),(1,0,1),(-1,0,1),(1,0,-1),(0,-1,-1),(0,1,1),(0,-1,1),(0,1,-1)]
n = idx.size
for bx,by,bz in [(16,1,1),(8,2,1),(4,4,1),(4,2,2),(2,4,2),(8,1,2),(4,1,1),(2,2,2),(4,2,1)]:
    px=(-nx)%bx
    a=np.pad(nd,((0,0),(0,0),(0,px)),constant_values=True)
    Z,Y,X=a.shape
    listed = ~a.reshape(Z//bz,bz,Y//by,by,X//bx,bx).all(axis=(1,3,5))
    lf = listed.mean()*listed.size*bx*by*bz/n
    # reads: per direction, bricks touched by shifted listed bricks (cell-level shift by 1 -> brick dilation in the nonzero comps)
    reads=0
    for cx,cy,cz in D:
        t=listed.copy()
        # source cells = dest - c: a dest brick touches bricks b and b - sign(c) along each nonzero axis
        if cx: t = t | np.roll(t, -int(np.sign(cx)) if False else 0, axis=2)
        tt=listed.copy()
        for ax,c in ((2,cx),(1,cy),(0,cz)):
            if c: tt = tt | np.roll(tt, shift=-c, axis=ax)
        reads += tt.sum()
    lines_per_cell_read = reads*128/ (n) 
    writes = listed.sum()*19*128/n
    print(f"brick {bx}x{by}x{bz}: listed cell frac {lf:.3f}  reads {reads*128/1e9:.1f} GB  writes {listed.sum()*19*128/1e9:.1f} GB  total {(reads+listed.sum()*19)*128/1e9:.1f} GB")
