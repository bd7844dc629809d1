"""B200-native (sm_100a, fp64) EBG tensor hyper-diffusion and Euler RHS.

From-scratch re-implementation of the hot path of arXiv 2311.11425's HEVI
spectral-element solver (reference package ``hevicore``) behind the
reference's own Python operator entry points:

* ``mesh``      -- MeshConfig / Mesh / build_box / build_cubed_sphere (host C++ numbering)
* ``metrics``   -- curl-invariant / cross-product metrics, column projection (device)
* ``assembly``  -- weights3 / gather / dss / GlobalMass (device)
* ``hyperdiff`` -- HyperDiffConfig / build_viscous_metric / laplacian_apply / hyperdiffusion_apply
* ``euler``     -- EulerOps (rhs_full / rhs_horizontal / hyper-diffusion plan)
* ``state``     -- PhysConstants / StateField / pressure

All numerics run in the C-ABI library ``libhv_b200.so`` (include/hv_b200.h);
there is no CPU fallback.
"""

__version__ = "0.1.0"
