import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, golden_io as G
from paper_2008_00326_b200.engine import default_engine
from paper_2008_00326_b200 import colorspace
U=G.load("units"); e=default_engine(); p=U["ciede_pairs"]
de=e.ciede2000(p[:,0:3],p[:,3:6]); h=colorspace.ciede2000(p[:,0:3],p[:,3:6])
for i in range(len(p)):
    if abs(de[i]-p[i,6])>1e-4 or abs(de[i]-h[i])>1e-9: print(i,p[i],de[i],h[i])
