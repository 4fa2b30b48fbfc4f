import sys; sys.path.insert(0, '.')
import paper_2504_03074_b200 as wh
g = wh.build_grid(2, [(0.0, 1.0)] * 2, [128, 128], "dirichlet")
dp = wh.device.device_problem(g)
print("plan", dp.ctx.plan())
