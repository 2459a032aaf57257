"""CPU oracle for the neural-preconditioned FGMRES hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2505_08491_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker (or the timed CPU baseline), never as the thing measured on the GPU.

It restates the reference algorithm (``/root/reference/pkg/src/mdprec``,
cited per function as ``file:line``) in numpy / scipy, float64 throughout,
plus the BASELINE.json semantics the reference cannot express directly
(SURVEY.md Appendix A): decoupled coupling weight beta, fixed elements per
edge, homogeneous Dirichlet on the cube, the seeded random-tree generator,
the nodal 1D load and the relaxed radius check for config 4.

Parity is pinned: ``tests/golden/make_golden.py`` imports the reference in
the build container and dumps fixtures that ``tests/test_oracle_golden.py``
checks this restatement against (bit-exact indices, <=1e-13 values,
identical FGMRES iteration counts).
"""

from .problem import (  # noqa: F401
    StructuredGrid, Graph, GraphMesh, PhysicalParams, CoupledSystem,
    refine_graph, random_tree, segment_graph, distance_field,
    trilinear_eval_matrix, build_restriction, assemble_coupled_system,
    full_operator, reduced_operator, one_d_operator, full_rhs, reduced_rhs,
    assemble_3d,
)
from .solver import (  # noqa: F401
    SolveReport, fgmres, ilu0, ilu0_apply, jacobi_smooth,
)
from .unet import (  # noqa: F401
    ARCHITECTURE, init_unet_params, noisy_params, unet_forward, conv3d,
    transposed_conv3d, maxpool3d, apply_neural, apply_batched,
    save_checkpoint, load_checkpoint, forward_flops,
)
from .coupled import solve_coupled, CoupledStrategy  # noqa: F401
