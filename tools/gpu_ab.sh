timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import bench
from paper_2604_01844_b200 import gsct
ctx = gsct.context(0); ctx.set_async(True)
for _ in range(3): print(bench.secondary_train(ctx, 5)['ms_per_iteration'])
"
