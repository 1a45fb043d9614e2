"""One K-best call at B=16, N=512, C=64 (a latency-bound shape) for ncu.  argv: K S"""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_00876_b200 as tsb, tsgen
K, S = int(sys.argv[1]), int(sys.argv[2])
pot = torch.empty((16, 511, 64, 64), dtype=torch.float32, device="cuda:0")
tsgen.fill_torch(pot, 11)
tsb.set_kbest_split(S)
tsb.kbest(pot, K); torch.cuda.synchronize()
