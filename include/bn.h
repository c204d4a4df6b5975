/*
 * bn.h — C ABI of the B200-native batched midsize-integer library (libbn.so).
 *
 * Implements the data-parallel hot path of Oancea & Watt, "GPU
 * Implementations for Midsize Integer Addition and Multiplication"
 * (arXiv 2405.14642; PAPER.md = /root/reference/PAPER.md at build time):
 * batches of fixed-width unsigned integers, one instance (or a few) per CTA,
 * sm_100a only.  No CUDA or torch types appear in the signatures.
 *
 * REPRESENTATION (§2): an integer is M little-endian limbs
 * A = sum_i a_i x^i, x = 2^(limb_bits); "the result has the same length and
 * element type as the input integers".  A batch is instance-major and
 * contiguous: instance k occupies limbs [k*n_limbs, (k+1)*n_limbs).
 * limb_bits = 64 is accepted and is the same bytes as 2*n_limbs u32 limbs
 * (little-endian device), so every kernel works on u32 limbs internally.
 *
 * SIZES: bits = n_limbs * limb_bits must be a power of two in
 * [1024, bn_op_max_bits(op)].  Every operation covers [1024, 262144] (the
 * paper's 2^11..2^18 sweep, PAPER.md:919 and Tables 1-2, plus 2^10), one
 * instance (or several) per CTA: 262144 bits is the largest size whose exact
 * NTT product fits one CTA's shared memory.  bn_add and bn_mul_ntt go on to
 * 2^19 and 2^20 bits, bn_mul_classical to 2^19, with one instance per
 * thread-block cluster of 2 / 4 CTAs (carries, NTT exchanges and the L/H
 * publish through distributed shared memory);
 * the fused (6-Add, Poly) and wide products stop at 2^18.  Other sizes ->
 * BN_ESIZE.
 *
 * POINTERS: a, b, out are DEVICE pointers on the current CUDA device, 16-byte
 * aligned.  out may equal a or b exactly (in-place); a partial overlap is
 * rejected.  The caller owns every buffer; the library owns only immutable
 * per-device NTT constant tables (freed at process exit).
 *
 * STREAMS: every call is stream-ordered and asynchronous on `stream`
 * (a cudaStream_t; NULL = legacy default stream), performs no allocation and
 * no host synchronisation — once the device is initialised.  The FIRST call
 * of any entry point on a device initialises it (bn_prepare: one cudaMalloc
 * of the NTT tables and synchronous uploads), so call bn_prepare(device)
 * up front when the first call must be asynchronous or is made under
 * CUDA-graph stream capture (an initialising call inside a capture fails).
 *
 * ALIASING AND ORDER: in-place calls are safe because every CTA reads all
 * of an instance's limbs before any write to that instance, and only the
 * thread that read a limb (add) or the CTA that staged the instance (mul)
 * writes it; the kernels therefore do not declare out / a / b __restrict__.
 *
 * ERRORS: argument errors return synchronously before any launch and write
 * nothing; a failed launch returns BN_ECUDA (see bn_cuda_error()); device
 * faults surface at the caller's next synchronisation.  n_inst == 0 returns
 * BN_OK without launching.
 */
#ifndef BN_H_
#define BN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *bn_stream_t; /* == cudaStream_t */

typedef enum {
    BN_OK = 0,
    BN_EINVAL = 1, /* NULL pointer, limb_bits not 32/64, n_limbs == 0, bad op */
    BN_ESIZE = 2,  /* n_limbs*limb_bits not a power of two in [1024, bn_op_max_bits(op)] */
    BN_EALIGN = 3, /* a, b or out not 16-byte aligned */
    BN_EALIAS = 4, /* out partially overlaps a or b (exact equality allowed) */
    BN_ECUDA = 5,  /* CUDA launch / configuration / copy failure */
    BN_ENODEV = 6  /* no usable device: the library holds sm_100a code only (CC 10.0) */
} bn_status;

/*
 * bn_add — out[k] = (a[k] + b[k]) mod 2^bits, k in [0, n_inst).
 * PAPER.md:144-163 (§2: map -> exclusive carry scan -> map), the carry
 * operator of PAPER.md:177-205 / Fig. 3 (carry_op_eff), batched as bbadd
 * (PAPER.md:232-234).  Each instance's carry-in is zero and its top carry-out
 * is dropped (fixed width; reading R1/R4).
 */
bn_status bn_add(void *out, const void *a, const void *b, uint64_t n_inst,
                 uint32_t n_limbs, uint32_t limb_bits, bn_stream_t stream);

/*
 * bn_mul_classical — out[k] = (a[k] * b[k]) mod 2^bits by the quadratic
 * algorithm: Eq. (1) with the load-balanced result
 * partitioning of Fig. 5, per-thread convolution and
 * L/H publish of Figs. 6-7, carries resolved by the
 * addition above.
 */
bn_status bn_mul_classical(void *out, const void *a, const void *b, uint64_t n_inst,
                           uint32_t n_limbs, uint32_t limb_bits, bn_stream_t stream);

/*
 * bn_mul_ntt — out[k] = (a[k] * b[k]) mod 2^bits by number-theoretic
 * transform over word-size primes p = k*2^n + 1 (§4).
 * Exact variant (readings R10/R11): 32-bit limbs are the digits,
 * zero-padded to N = 2*n_limbs32 points, three primes < 2^30 and Garner CRT,
 * Shoup/Montgomery modular arithmetic ("further improvement
 * would be expected using Montgomery representation").  Results are
 * bit-identical to bn_mul_classical.  Builds the constant tables on first use
 * on a device (bn_prepare), which synchronises once.
 */
bn_status bn_mul_ntt(void *out, const void *a, const void *b, uint64_t n_inst,
                     uint32_t n_limbs, uint32_t limb_bits, bn_stream_t stream);

/* ---- fused workloads (block-level fusion) ---------------
 * The paper's 6-Add and Poly benchmarks (Tables 1 and 2): several dependent
 * operations per instance inside ONE kernel, intermediates kept on chip (or,
 * for Poly, in a small per-CTA workspace that stays in L2), so that a batch
 * reads a and b once and writes one result ("both programs read two
 * integers from global memory and write one as result"
 * footnote).  Same layout, sizes, alignment, aliasing, stream and error
 * rules as bn_add.
 *
 * bn_add6 — out[k] = (4 a[k] + 3 b[k]) mod 2^bits computed as six dependent
 * scan-additions r = a + b, r += a, r += b, r += a, r += b, r += a (6-Add,
 * PAPER.md:917-918; the paper does not print the expression: DESIGN.md
 * reading R17).
 */
bn_status bn_add6(void *out, const void *a, const void *b, uint64_t n_inst,
                  uint32_t n_limbs, uint32_t limb_bits, bn_stream_t stream);

/*
 * bn_poly_classical / bn_poly_ntt — out[k] = ((a a + b)(b b + b) + a b)
 * mod 2^bits (Poly, PAPER.md:918 and the Table 2 caption: "four
 * multiplications and two additions"; the expression has three, all are
 * computed — DESIGN.md reading R18), with every multiplication done by the
 * classical (bn_mul_classical) or NTT (bn_mul_ntt) algorithm and each
 * addition fused into the epilogue of the product before it.
 * workspace: DEVICE buffer of at least bn_poly_workspace_bytes(op, n_inst,
 * n_limbs, limb_bits) bytes on the current device, 16-byte aligned, owned
 * by the caller, not overlapping a, b or out; its contents are scratch
 * (undefined after the call) and it must not be used by another call that
 * may run concurrently.  Too small -> BN_EINVAL, nothing launched.
 */
bn_status bn_poly_classical(void *out, const void *a, const void *b, uint64_t n_inst,
                            uint32_t n_limbs, uint32_t limb_bits, void *workspace,
                            uint64_t workspace_bytes, bn_stream_t stream);
bn_status bn_poly_ntt(void *out, const void *a, const void *b, uint64_t n_inst,
                      uint32_t n_limbs, uint32_t limb_bits, void *workspace,
                      uint64_t workspace_bytes, bn_stream_t stream);

/* ---- addition beyond one cluster ------------------------
 * bn_add_big — out[k] = (a[k] + b[k]) mod 2^bits, like bn_add, for any
 * power-of-two size from 2^18 to 2^30 bits, with the single-pass
 * decoupled look-back carry scan the paper's scan citation refers to
 * (PAPER.md:66, 289-292): every instance is cut into fixed-size tiles (at
 * most 2^18 bits; bn_config.h), one CTA per tile, tiles taken in order from
 * an atomic counter; each tile
 * publishes its carry aggregate, looks back over its predecessors' flags for
 * its carry-in, and publishes its carry-out.  Same layout,
 * alignment, aliasing and stream rules as bn_add; the number of tiles must
 * be < 2^31 (else BN_ESIZE).
 * workspace: DEVICE buffer of at least bn_add_big_workspace_bytes(...) bytes
 * (one 32-bit flag per tile + a counter), 16-byte aligned, owned by the
 * caller, not overlapping a, b or out, not shared with a concurrent call;
 * the call zeroes it on `stream` (cudaMemsetAsync) before the kernel.
 * Too small -> BN_EINVAL. */
bn_status bn_add_big(void *out, const void *a, const void *b, uint64_t n_inst, uint32_t n_limbs,
                     uint32_t limb_bits, void *workspace, uint64_t workspace_bytes, bn_stream_t stream);
/* Workspace bytes bn_add_big needs; 0 for n_inst == 0 or an invalid size. */
uint64_t bn_add_big_workspace_bytes(uint64_t n_inst, uint32_t n_limbs, uint32_t limb_bits);

/* Workspace bytes a bn_poly_* call needs on the CURRENT device for this
 * batch (one slice of 3 intermediates per resident CTA; <= 3 * n_inst *
 * bits / 8).  op = BN_OP_POLY_CLASSICAL or BN_OP_POLY_NTT.  Returns 0 for
 * n_inst == 0 or invalid arguments.  May initialise the device (bn_prepare). */
uint64_t bn_poly_workspace_bytes(int op, uint64_t n_inst, uint32_t n_limbs, uint32_t limb_bits);

/* ---- full (untruncated) products -------------------------
 * bn_mul_wide_classical / bn_mul_wide_ntt — out[k] = a[k] * b[k] exactly, as
 * 2*n_limbs limbs of limb_bits (Eq. 1, without the k < M
 * truncation: all columns 0 <= k < 2M).  out holds n_inst * 2 * n_limbs
 * limbs and may not overlap a or b at all (it is twice their size); a and b
 * follow bn_add's rules.  Classical: the truncated kernel's partition for
 * the low half and the same convolution on mirrored operands for the high
 * half; bits in [1024, 262144].  NTT: the N = 2m point
 * transforms already produce every coefficient; bits in [1024, 262144]
 * (at 262144 bits one 512-thread CTA per instance with a single exchange
 * plane and an incremental, element-wise Garner). */
bn_status bn_mul_wide_classical(void *out, const void *a, const void *b, uint64_t n_inst,
                                uint32_t n_limbs, uint32_t limb_bits, bn_stream_t stream);
bn_status bn_mul_wide_ntt(void *out, const void *a, const void *b, uint64_t n_inst,
                          uint32_t n_limbs, uint32_t limb_bits, bn_stream_t stream);

/* Initialise `device`: check it is CC 10.0 (else BN_ENODEV), build the NTT
 * twiddle/CRT tables (all sizes) and upload them, synchronously.  Idempotent
 * and thread-safe; every other entry point calls it lazily on first use. */
bn_status bn_prepare(int device);

/* ---- host-buffer entry point (end-to-end path) ---------------------------
 * bn_run_host — runs a sequence of operations over HOST operands: the batch
 * is cut into chunks that are copied host->device, processed by each op in
 * `ops` (same operands a, b), and copied device->host into outs[i], with
 * copies and kernels overlapped on three streams of the current device.
 * ops[i] is one of the BN_OP_* codes below (Poly ops get their workspace
 * from the pipeline's own scratch);
 * outs[i] is a host buffer of n_inst*n_limbs limbs.  Host buffers should be
 * page-locked (cudaHostAlloc / torch pin_memory) for full bandwidth.
 * Device scratch is allocated on first use and cached per device (grown on
 * demand).  Synchronous: returns when every output is in host memory. */
enum { BN_OP_ADD = 0, BN_OP_MUL_CLASSICAL = 1, BN_OP_MUL_NTT = 2, BN_OP_ADD6 = 3,
       BN_OP_POLY_CLASSICAL = 4, BN_OP_POLY_NTT = 5,
       /* not accepted by bn_run_host (output is twice the size); used by
        * bn_launches_per_call */
       BN_OP_MUL_WIDE_CLASSICAL = 6, BN_OP_MUL_WIDE_NTT = 7 };
bn_status bn_run_host(const int *ops, void *const *outs, int n_ops, const void *a,
                      const void *b, uint64_t n_inst, uint32_t n_limbs, uint32_t limb_bits);

/* ---- introspection ------------------------------------------------------ */
uint32_t bn_max_bits(void);                /* 1048576: the largest size any op accepts */
uint32_t bn_op_max_bits(int op);           /* per BN_OP_* code; 0 for an unknown op */
uint32_t bn_min_bits(void);                /* 1024 */
int bn_cuda_error(void);                   /* last cudaError_t seen by this thread */
const char *bn_status_string(bn_status s); /* static string */
/* Number of kernel launches one call of `op` makes at this size (>= 1), for
 * launch accounting in the benchmark; 0 for an unsupported size/op. */
uint32_t bn_launches_per_call(int op, uint32_t bits);

/* ---- NTT introspection / debug (tests only; not on the hot path) --------
 * bn_ntt_primes — writes the three primes used by bn_mul_ntt to p[0..2].
 * bn_debug_ntt_forward — x (device, n_inst*N u32 residues < p) -> forward
 * transform of each length-N row over prime index `prime` (0..2), in place,
 * output in BIT-REVERSED order and in [0, p), with omega_N = the library's
 * primitive N-th root for that prime, written to *omega_out.  N = 2^lg_n,
 * lg_n in [6, 14]. */
void bn_ntt_primes(uint32_t p[3]);
/* bn_debug_set_grid_cap — tests only: cap every kernel's grid at `cap` CTAs
 * (0 = default sizing) so small batches exercise the persistent /
 * grid-stride paths; results must not change (reading R20).
 * Process-wide, not thread-safe. */
void bn_debug_set_grid_cap(uint32_t cap);
bn_status bn_debug_ntt_forward(uint32_t *x, uint64_t n_inst, uint32_t lg_n, int prime,
                               uint32_t *omega_out, bn_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* BN_H_ */
