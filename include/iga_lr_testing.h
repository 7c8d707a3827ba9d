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
 * Results agree to rounding across all settings.  The call mutates the op: it must not run
 * concurrently with applies on the same op.  Errors: IGA_EINVAL (NULL, qx not in {0,1,2,4},
 * minlen < 0).
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
} iga_test_knobs;

iga_status iga_lr_test_knobs(iga_lr_op* op, const iga_test_knobs* k);

#ifdef __cplusplus
}
#endif
#endif /* IGA_LR_TESTING_H */
