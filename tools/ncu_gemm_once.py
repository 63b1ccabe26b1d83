import sys; sys.path.insert(0,'.')
from paper_2111_11728_b200 import engine
engine.dla_time_gemm(2048,2048,4096,False,False,reps=1)
