// apply_fused2.cu — fused v2 / canonical-shape kernels: host side, generic v2 kernel, fixup.
// (implementation in fused2_impl.cuh; per-degree kernel instantiations in canon_p3.cu, canon_p4.cu)
#include "fused2_impl.cuh"
