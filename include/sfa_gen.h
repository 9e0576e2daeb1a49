/*
 * include/sfa_gen.h -- device side of the seeded synthetic-input generator.
 *
 * Not part of the method: it only draws the dense Q, K, V the method consumes, bit-identical
 * to paper_2603_22300_b200/inputs.py (the host side, used by the oracle tests), so large
 * inputs (32K-1M tokens) can be created in HBM while the oracle regenerates sampled rows
 * on the host.  Recipe in inputs.py / DESIGN.md "Input recipe".
 */
#ifndef SFA_GEN_H
#define SFA_GEN_H
#include <stdint.h>
#include "sfa.h"
#ifdef __cplusplus
extern "C" {
#endif

typedef enum { SFA_GEN_IID = 0, SFA_GEN_LATTICE = 1, SFA_GEN_SKEWED = 2 } sfa_gen_variant;

/* out[i] for flat index i in [offset, offset + count) of a tensor shaped [..., n, d]
 * (n, d only matter for SFA_GEN_SKEWED, whose gain is per (head, feature)).
 * out is a DEVICE pointer to `count` elements of `dtype`.  Stream-ordered. */
SFA_API sfa_status sfa_gen_fill(void *out, sfa_dtype dtype, int64_t count, int64_t offset, uint64_t seed, int32_t tensor_id,
                        int32_t variant, int64_t n, int32_t d, int32_t skew_span, sfa_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
