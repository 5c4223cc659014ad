/*
 * qflash_debug.h -- bring-up entry point of libqflash.so (not part of the
 * production ABI; used by tests/test_gpu_parity.py to localise a mismatch).
 */
#ifndef QFLASH_DEBUG_H_
#define QFLASH_DEBUG_H_

#include "qflash.h"

#ifdef __cplusplus
extern "C" {
#endif

/* qflash_attention_int8_ex with host scales, plus raw dumps from the CTA that
 * owns (problem 0, query tile 0), each device int32, may be NULL:
 *   dbg_s [128][B_c]     S = Q K_0^T of KV tile 0 (step 1), TMEM lane = row
 *   dbg_p [128][B_c/4]   packed int8 P of KV tile 0 (steps 5-6), byte i = key 4w+i
 *   dbg_o [128][d+1]     final O accumulator and l (last column) before step 11
 *   dbg_t [128] int64    clock64() timeline of that CTA (slots in qflash_attention.cu)
 * (For the packed variant B_c = 128: two 64-key windows.) */
QFLASH_API qflash_status qflash_debug_attention(const int8_t* q, const int8_t* k, const int8_t* v,
                                                float s_q, float s_k,
                                                const qflash_attn_shape* shape,
                                                qflash_variant variant, int8_t* o, int32_t* dbg_s,
                                                int32_t* dbg_p, int32_t* dbg_o, long long* dbg_t,
                                                qflash_stream_t stream);

/* Force the attention kernel configuration of every later launch in this process
 * (tests and A/B runs; the host heuristic picks one otherwise):
 *   cfg -1  the heuristic (default; QFLASH_ATTN_CFG=<0..3> in the environment sets
 *           the initial value)
 *   cfg 0   CS = 4 column splits x QT = 1 query tile in flight
 *   cfg 1   CS = 2 x QT = 2
 *   cfg 2   row-owner softmax + correction warpgroups x QT = 2
 *   cfg 3   row-owner softmax + correction warpgroups x QT = 1
 * A forced configuration that has no instantiation for a shape (TMEM / shared
 * memory budget) falls back to the heuristic's choice.  Returns
 * QFLASH_ERR_INVALID_ARGUMENT for cfg outside [-1, 3].  Not thread-safe with
 * respect to launches already being prepared on other threads. */
QFLASH_API qflash_status qflash_debug_force_config(int32_t cfg);

/* The configuration (bits 0-3) and row-packing segment count NSEG (bits 4-7) of
 * the calling thread's last attention launch, or -1 if it made none. */
QFLASH_API int32_t qflash_debug_last_config(void);

#ifdef __cplusplus
}
#endif

#endif /* QFLASH_DEBUG_H_ */
