"""paper_1911_09135_b200 — B200-native ALB (adaptive load balancer) graph analytics.

Drop-in for the reference ``simtgraph`` package's hot path (engine.run /
run_app with bfs, sssp, cc, pr, kcore; Graph / generate_rmat /
attach_random_weights; the kernel-backend plugin protocol), executing on
hand-written sm_100a CUDA kernels through libsimtgraph_cuda.so.

    import paper_1911_09135_b200 as simtgraph
    g = simtgraph.graph.generate_rmat(20, 16, 1)
    r = simtgraph.engine.run_app(g, "bfs", simtgraph.schedulers.Scheduler("alb"))
"""

from . import apps, engine, errors, graph, kernels, schedulers, simt  # noqa: F401
from .engine import report, run, run_app  # noqa: F401
from .graph import Graph, attach_random_weights, generate_rmat, load_graph  # noqa: F401
from .schedulers import Scheduler  # noqa: F401
from .simt import KernelConfig  # noqa: F401

__version__ = "0.1.0"
