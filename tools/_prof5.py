import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import bench_configs as bc
bc.cfg5(1, 0, B=int(sys.argv[1]) if len(sys.argv) > 1 else 512, tols=(1e-10,))
