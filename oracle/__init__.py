"""Oracle package — TEST INFRASTRUCTURE ONLY (see oracle/lsk_oracle.py header).

May be imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg.  Never by the product package paper_2006_07057_b200.
"""
from .lsk_oracle import *  # noqa: F401,F403
from .lsk_oracle import (lambert_w0, max_norm, gaussian_params, philox4x32_10, philox_words,
                         standard_normals, draw_anchors, gaussian_phi, feature_matrix,
                         feature_entries_scaled, sinkhorn, sinkhorn_factored, sinkhorn_dense,
                         dual_estimate, primal_objective, gaussian_kernel_dense,
                         marginal_error, rot, sinkhorn_divergence, envelope_gradients,
                         arccos_phi, arccos_kernel, feature_matrix_arccos)
