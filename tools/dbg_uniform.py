import sys, os, math
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1609_01277_b200 as osbli
from inputs import uniform_state
for shape, order in [((17,9,11),12), ((32,16,8),4), ((64,32,8),2)]:
    s = osbli.Solver(*shape, order, 0.3, 1e-3)
    s.set_state(uniform_state(*shape))
    R = s.residual()
    nz = [(f, np.abs(R[f]).max()) for f in range(5)]
    print(shape, order, nz)
    idx = np.argwhere(np.abs(R[4]) > 0)
    print(' nonzero count', len(idx), 'of', R[4].size, 'sample', idx[:5].tolist())
    s.set_state(uniform_state(*shape, u=(0,0,0)))
    R = s.residual(); print(' u=0:', [np.abs(R[f]).max() for f in range(5)])
