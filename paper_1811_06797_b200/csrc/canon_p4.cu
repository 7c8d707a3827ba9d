// canon_p4.cu — instantiations of the canonical fused kernel for degree 4 (parallel build unit).
#define IGALR_CANON_P 4
#include "fused2_impl.cuh"
