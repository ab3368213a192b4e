import sys,time; sys.path.insert(0,".")
import numpy as np
import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs
for idx in (3,5):
    c=configs.make_case(idx); px,py,pz=c.boxes
    t=time.time(); h=dk.subdomain_levelset_partition(c.band_field,px,py,pz,c.jump_threshold,backend="host"); th=time.time()-t
    for r in range(4):
        t=time.time(); d=dk.subdomain_levelset_partition(c.band_field,px,py,pz,c.jump_threshold,backend="device"); td=time.time()-t
        print(idx, r, d.d, h.d, int((d.labels!=h.labels).sum()), f"dev {td:.3f}s host {th:.3f}s")
