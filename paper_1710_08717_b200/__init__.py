"""paper_1710_08717_b200 — B200-native (sm_100a) batched differentiable dense
linear algebra: the reference dlinalg operator layer (potrf / potri / trsm /
trmm / gemm / gemm2 / syrk / sumlogdiag / gelqf / syevd, forward and
closed-form backward, f32/f64) behind a C-ABI (include/dla.h,
libdla_b200.so).  See DESIGN.md.

``linalg`` is the reference-facing API; ``gp`` the GP NLL driver; ``shard``
the multi-GPU batch sharder.  Importing ``linalg`` loads libdla_b200.so and
fails loudly if it is missing — there is no CPU fallback.
"""
__version__ = "0.1.0"
