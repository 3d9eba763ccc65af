"""Small fused-MLP solve (debug helper for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2210_12375_b200 as bode
z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "mlp.npz"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
backend = sys.argv[2] if len(sys.argv) > 2 else "fused"
y0 = np.random.default_rng(0).normal(size=(n, 64))
prob = bode.IvpBatch(y0, np.zeros(n), np.full(n, 2.0), np.full((n, 1), 2.0))
sol = bode.solve(prob, bode.mlp_dynamics(z["W1"], z["b1"], z["W2"], z["b2"]), max_steps=1000,
                 mlp_backend=backend)
print(backend, "status", np.bincount(sol.status), "steps", sol.stats.n_steps.sum(), "ys0", sol.ys_flat[0, :3])
