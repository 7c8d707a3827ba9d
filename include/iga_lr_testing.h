/*
 * iga_lr_testing.h — TEST-ONLY entry point of libigalr.so (not part of the product API in
 * iga_lr.h; the product never reads environment variables to pick kernels).
 *
 * iga_lr_test_knobs overrides the kernel-selection choices of ONE op so that tests and
 * experiments can reach every kernel variant:
 *   force_generic : != 0 => fused-v2 parts run the generic k_fused2 even when the plan has
 *                   the canonical shape (and the KKT skips its canonical launches)
 *   qx            : 0 (auto) or 1/2/4 => canonical tiles of 32*qx columns
 *   minlen        : 0 (auto) or > 0 => persistent-CTA ranges of `minlen` z-planes
 *   no_yres       : != 0 => per-round y-coefficient staging instead of resident tables
 *   no_tma        : != 0 => no bulk-copy (cp.async.bulk) staging
 *   vpack         : 0 (auto) or > 0 => canonical tiles hold `vpack` vectors side by side along x
 *                   (1: no packing; clamped to the batch; bulk-copy path only)
 * Results agree to rounding across all settings.  The call mutates the op: it must not run
 * concurrently with applies on the same op.  Errors: IGA_EINVAL (NULL, qx not in {0,1,2,4},
 * minlen < 0, vpack < 0).
 */
#ifndef IGA_LR_TESTING_H
#define IGA_LR_TESTING_H

#include "iga_lr.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t force_generic;
    int32_t qx;
    int32_t minlen;
    int32_t no_yres;
    int32_t no_tma;
    int32_t vpack;
} iga_test_knobs;

iga_status iga_lr_test_knobs(iga_lr_op* op, const iga_test_knobs* k);

/*
 * iga_lr_test_tile reports the canonical tile the library picks for a launch over `batch` vectors
 * (knobs included): tiles of 32*qx columns and 2*lw*(4/qx) rows, and vp vectors packed side by side
 * along x (vp = 1: no packing).  Errors: IGA_EINVAL (NULL, batch < 1),
 * IGA_EUNSUPPORTED (no canonical kernel for the op's degree).
 */
iga_status iga_lr_test_tile(const iga_lr_op* op, int32_t batch, int32_t* qx, int32_t* lw, int32_t* vp);

#ifdef __cplusplus
}
#endif
#endif /* IGA_LR_TESTING_H */
