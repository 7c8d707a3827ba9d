// canon_p3.cu — instantiations of the canonical fused kernel for degree 3 (parallel build unit).
#define IGALR_CANON_P 3
#include "fused2_impl.cuh"
