import sys
sys.path.insert(0, '.')
sys.argv=['x']
import tools.gemm_bw as G
for M,K in ((4096,4096),(28672,4096),(4096,14336)):
    for rows in (16,32,64,128,256):
        G.run(M,K,rows)
