"""Line-granular DRAM model of the compacted porous sweep (k_cmp) at the c4
bench geometry: distinct 32-B sectors / 64-B pairs / 128-B lines read per
pull direction over the compact arrays (profiles/r02b_summary.md).

    python tools/c4_line_model.py [L]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09242_b200 as dlb
L=int(sys.argv[1]) if len(sys.argv)>1 else 600
cfg = dlb.CaseConfig(kind="porous", L=L, Ma=0.01, collision=dlb.LinkType.TRT, q=19, tau=1.0, upstream=40, downstream=40)
vox, phi = dlb.sphere_pack((L, L, L), radius=8.0, porosity=0.20, seed=20250611)
setup = dlb.init_porous(cfg, solid=(vox == 255))
idx = np.asarray(setup.chain_index); nz,ny,nx = idx.shape
G=4; nsx=(nx+G-1)//G
nd = np.pad(idx==2, ((0,0),(0,0),(0,nsx*G-nx)), constant_values=True)
listed = ~nd.reshape(nz,ny,nsx,G).all(-1)       # (z,y,s) interior
# extended grid with envelope segments s=-1..nsx, rows periodic in y,z (porous case) -> no envelope rows needed
E = np.zeros((nz,ny,nsx+2),bool); E[:,:,1:-1]=listed
D=[(0,0,0),(-1,0,0),(1,0,0),(0,-1,0),(0,1,0),(0,0,-1),(0,0,1),(-1,-1,0),(1,1,0),(-1,1,0),(1,-1,0),(-1,0,-1),(1,0,1),(-1,0,1),(1,0,-1),(0,-1,-1),(0,1,1),(0,-1,1),(0,1,-1)]
inset = E.copy()
for cx,cy,cz in D:
    # dest (z,y,s) pulls from row (y-cy, z-cz): source row = roll of dest by (+cz? ) : src[z-cz,y-cy] <- dest[z,y]
    t = np.roll(E, shift=(-cz,-cy), axis=(0,1))  # t[Z,Y] = E[Z+cz, Y+cy] = dest at row whose source is (Z,Y)
    inset |= t
    if cx>0: inset[:,:,:-1] |= t[:,:,1:]
    if cx<0: inset[:,:,1:] |= t[:,:,:-1]
flat = inset.reshape(-1)
cidx = np.cumsum(flat)-1
ncomp = flat.sum(); nl = listed.sum()
print("listed segs", nl, "compact segs", ncomp, "ratio", ncomp/nl)
# per direction: sectors touched: for dest listed seg with compact index m_src(row', s): cells m*4+lane-cx for lane 0..3
tot32=0; tot64=0; tot128=0
Ei = np.where(E.reshape(-1))[0]  # dest ids in extended grid
for cx,cy,cz in D:
    srcE = np.roll(np.arange(E.size).reshape(E.shape), shift=(cz,cy), axis=(0,1)).reshape(-1)  # srcE[dest] = id of (z-cz,y-cy,s)
    m = cidx[srcE[Ei]]
    cells = (m[:,None]*4 + np.arange(4)[None,:] - cx).reshape(-1)
    s32 = np.unique(cells//4); s64=np.unique(cells//8); s128=np.unique(cells//16)
    tot32+=len(s32); tot64+=len(s64); tot128+=len(s128)
print("read sectors per listed seg: 32B %.2f  64B-pairs*2 %.2f  128B-lines*4 %.2f" % (tot32/nl, 2*tot64/nl, 4*tot128/nl))
print("GB at 32B: %.2f, 64B: %.2f, 128B: %.2f" % (tot32*32/1e9, tot64*64/1e9, tot128*128/1e9))
