"""Paper Listings 1-4: 2D diffusion on a 4x4 grid, written
exactly as in the paper, decomposed over however many ranks launch it.

    python examples/listing4_diffusion.py
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 examples/listing4_diffusion.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2312_13094_b200 import Eq, Grid, Operator, TimeFunction, solve  # noqa: E402

nx, ny = 4, 4
grid = Grid(shape=(nx, ny), extent=(2.0, 2.0))
u = TimeFunction(name="u", grid=grid, space_order=2)
u.data[1:-1, 1:-1] = 1                      # logically global write (Listing 1)
print(f"rank {grid.ctx.rank}: local view\n{u.data[:]}")   # per-rank views (Listing 3)
op = Operator([Eq(u.forward, solve(Eq(u.dt, u.laplace), u.forward))])
dx = 2.0 / (nx - 1)
op.apply(time_M=1, dt=0.25 * dx * dx / 0.5, mpi=os.environ.get("STENCIL_DMP_MODE", "full"))
g = u.data_gather()
if grid.ctx.rank == 0:
    print("after 2 steps (Listing 4):\n", g)
