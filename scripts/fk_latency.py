import sys; sys.path.insert(0, "/root/repo")
import paper_2005_07068_b200 as hp, workloads as W
ctx = hp.Context(640, 480, max_particles=64)
for i in range(3): ctx.debug_fk(W.H_A)
