/*
 * dsv.h — C ABI of the B200 state-vector engine (libdsv.so).
 *
 * The reference (`duetsim`, /root/reference/pkg/src/duetsim) has no FFI: its
 * hot path is a set of module-level NumPy "raw kernels" that mutate a
 * caller-owned amplitude array in place, addressed by PHYSICAL index bits.
 * Every entry point below replaces one of those functions (or one
 * StateVector / SegmentedStateVector primitive built on them); the cited
 * file:line is the reference interface it stands in for.
 *
 * Conventions
 *  - A `dsv_state` is one contiguous 2^nbits amplitude segment resident in
 *    HBM on one device (the whole vector for StateVector, one segment for
 *    SegmentedStateVector / the multi-GPU layer).  Amplitudes are interleaved
 *    (re, im) float32 (DSV_C64) or float64 (DSV_C128), little-endian index:
 *    bit b of an index is index bit b (statevec.py module doc, core.py:3-5).
 *  - Gate data (matrices, diagonals) is passed in the STATE dtype, as the
 *    reference's StateVector casts it (statevec.py:181, :191).  Host pointers
 *    are borrowed for the duration of the call only.
 *  - Matrix index bit m <-> targets[m] (gates.py:3-5), row-major 2^k x 2^k.
 *  - Controls are (bit, value) pairs; value 0 is an anti-control.
 *  - Return value: 0 ok, 1 invalid argument, 2 CUDA error, 3 out of memory,
 *    4 unsupported.  dsv_last_error() returns the thread-local message.
 *  - Calls are stream-ordered on the state's private stream and return
 *    before the GPU finishes, except those that return host data (reductions,
 *    downloads, sampling), which synchronise.  A state must not be mutated
 *    concurrently from two host threads (SPEC.md:188-189 ownership rule).
 *  - There is no CPU fallback: with no usable CUDA device every call that
 *    touches a state returns 2.
 */
#ifndef DSV_H
#define DSV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSV_OK 0
#define DSV_EINVAL 1
#define DSV_ECUDA 2
#define DSV_ENOMEM 3
#define DSV_EUNSUPPORTED 4

#define DSV_C64 0
#define DSV_C128 1

#define DSV_MAX_TARGETS 10 /* fusion.py:22 _MAX_FUSED_QUBITS */
#define DSV_MAX_BITS 40

typedef struct dsv_state dsv_state;

/* ---- library / device ------------------------------------------------- */
const char* dsv_last_error(void);
int dsv_version(void);
int dsv_device_count(int* out);
/* Kernel-selection switches, otherwise read once from the environment:
 * "tc" (DSV_TC: tensor-core windows), "tc8" (DSV_TC8: int8-digit tcgen05
 * kernels; 0 selects the bf16-limb fp32-level tc.cu / tc6.cu), "low", "lowt",
 * "dblk8", "blk8", "wt".  Process-wide; takes effect for the next call. */
int dsv_config_set(const char* key, int value);
/* total number of this library's kernel launches so far (all states) */
int dsv_launch_count(uint64_t* out);

/* ---- lifecycle (statevec.py:122-128 StateVector.__init__, distsim.py:70-84) */
/* Allocate 2^nbits amplitudes on `device`, initialised to |0...0>. */
/* Destroyed states park their device buffer in a small per-process cache that
 * dsv_state_create reuses for the same (device, size); a failed allocation
 * empties it first.  This releases the cache (device < 0: all devices).
 * DSV_POOL=0 in the environment disables caching. */
int dsv_pool_release(int device);
int dsv_state_create(int device, int nbits, int dtype, dsv_state** out);
int dsv_state_destroy(dsv_state* s);
int dsv_state_info(const dsv_state* s, int* device, int* nbits, int* dtype);
/* raw device pointer of the segment (for IPC / tests) */
int dsv_state_device_ptr(const dsv_state* s, void** out);
int dsv_sync(dsv_state* s);

/* ---- data movement ------------------------------------------------------ */
/* |index> (statevec.py:126-127 sets amplitude 0 to 1; also used per segment) */
int dsv_set_basis(dsv_state* s, uint64_t index);
int dsv_set_zero(dsv_state* s);
/* physical-order copies of [begin, begin+count) to/from host */
int dsv_upload(dsv_state* s, uint64_t begin, uint64_t count, const void* host);
int dsv_download(dsv_state* s, uint64_t begin, uint64_t count, void* host);
/* device-to-device copy of a whole segment (statevec.py:156-161 copy) */
int dsv_copy(dsv_state* dst, const dsv_state* src);

/* ---- gate application: the hot path ------------------------------------ */
/* replaces apply_dense_bits, statevec.py:44-60 */
int dsv_apply_matrix(dsv_state* s, const void* matrix, const int32_t* targets, int k,
                     const int32_t* ctrl_bits, const int32_t* ctrl_vals, int nctrl);
/* replaces apply_permutation_bits, statevec.py:63-81:
 * out[perm[j]] = diag[j] * in[j] per control-satisfied group, complex product
 * in NumPy's FMA form (re = fma(dr, ar, -(di*ai)), im = fma(dr, ai, di*ar)). */
int dsv_apply_genperm(dsv_state* s, const int64_t* perm, const void* diag,
                      const int32_t* targets, int k, const int32_t* ctrl_bits,
                      const int32_t* ctrl_vals, int nctrl);
/* Fused window of the opt-in fold fuser (fusion_fold.py; extension of the
 * reference's fused gates, fusion.py:97-121): dense matrix on `targets`
 * applied after the diagonal exp(i (sum_x theta_x [target cross_t[x]] [bit cross_b[x]]
 * + sum_y out_theta[y] [bit out_b[y]])), cross_t indexing `targets`, cross_b /
 * out_b physical bits outside the targets.  k <= 5, no controls. */
int dsv_apply_matrix_phased(dsv_state* s, const void* matrix, const int32_t* targets, int k,
                            const int32_t* cross_t, const int32_t* cross_b, const double* cross_theta,
                            int ncross, const int32_t* out_b, const double* out_theta, int nout);
/* replaces StateVector.apply_pauli_rotation, statevec.py:196-207 (copy-free):
 * psi <- cos(theta/2) psi - i sin(theta/2) coef (P psi); paulis[i] in "IXYZ" */
int dsv_apply_pauli_rotation(dsv_state* s, double theta, double coef_re, double coef_im,
                             const int32_t* bits, const char* paulis, int m);
/* replaces apply_pauli_product_bits, statevec.py:84-104 (unit coefficient) */
int dsv_apply_pauli_product(dsv_state* s, const int32_t* bits, const char* paulis, int m);

/* ---- layout ------------------------------------------------------------ */
/* replaces StateVector.swap_index_bits data movement, statevec.py:311-324
 * (in place; pairs = 2*npairs ints, disjoint, validated by the caller as in
 * core.py:21-30; (b,b) is a no-op) */
int dsv_swap_index_bits(dsv_state* s, const int32_t* pairs, int npairs);
/* replaces StateVector.access, statevec.py:278-294: out[t] = amp[src(begin+t)],
 * src(j) = sum_b bit_b(j) << ordering[b] */
int dsv_access_get(dsv_state* s, const int32_t* ordering, uint64_t begin, uint64_t end,
                   void* host_out);
/* replaces StateVector.access_set, statevec.py:296-309 */
int dsv_access_set(dsv_state* s, const int32_t* ordering, uint64_t begin, uint64_t count,
                   const void* host_in);

/* ---- reductions (synchronising; float64 accumulation, fixed order) ------ */
/* replaces norm_squared, core.py:62-71 / statevec.py:153-154 */
int dsv_norm2(dsv_state* s, double* out);
/* replaces marginal_probabilities_bits, statevec.py:107-113: out[o], bit j of o
 * = value of bits[j] */
int dsv_marginal_probs(dsv_state* s, const int32_t* bits, int k, double* out);
/* replaces the Pauli branch of StateVector.expectation, statevec.py:246-253:
 * out = <psi| P |psi> (re, im) for one unit-coefficient Pauli string */
int dsv_expect_pauli(dsv_state* s, const int32_t* bits, const char* paulis, int m,
                     double* out_re_im);
/* replaces the DenseGate branch of StateVector.expectation, statevec.py:241-245 */
int dsv_expect_matrix(dsv_state* s, const void* matrix, const int32_t* targets, int k,
                      double* out_re_im);
/* <a|b> for two segments of equal shape (np.vdot) */
int dsv_inner(dsv_state* a, const dsv_state* b, double* out_re_im);
/* replaces the collapse step of StateVector.measure, statevec.py:229-237:
 * zero amplitudes whose `bits` disagree with `outcome`, scale the rest by
 * 1/sqrt(norm2_kept) */
int dsv_collapse(dsv_state* s, const int32_t* bits, int k, uint64_t outcome,
                 double norm2_kept);
/* scale every amplitude by a real factor (renormalisation helper) */
int dsv_scale(dsv_state* s, double factor);
/* replaces the CDF + searchsorted part of StateVector.sample, statevec.py:267-272:
 * outcomes[i] = first index whose cumulative |a|^2 exceeds variates[i]*total */
int dsv_sample(dsv_state* s, const double* variates, int64_t shots, uint64_t* outcomes);

/* ---- segments: global <-> local exchange (distsim.py:153-198) ---------- */
/* For every offset `off` with bit `local_bit` clear, swap
 *     a[off | 1<<local_bit]  <->  b[off]
 * i.e. the (global, local) index-bit swap between segment a (global bit 0)
 * and segment b (global bit 1), done in place in one pass.  The 2^(nbits-1)
 * offsets are split into `nparts` equal slices and this call performs slice
 * `part` (two processes owning a and b each run one half; nparts=1: all).
 * b may live on another device (peer access) or be a peer IPC mapping. */
int dsv_exchange_halves(dsv_state* a, dsv_state* b, int local_bit, int part, int nparts);
/* whole-segment swap a <-> b (global-global pairs when both differ) */
int dsv_exchange_all(dsv_state* a, dsv_state* b);

/* Batched (global, local) index-bit swaps between two segments
 * (distsim.py:153-198 with q global bits at once): for every offset `off`
 * whose q local bits `lbits` are clear,
 *     a[off | pat_a]  <->  b[off | pat_b]
 * where pat_a / pat_b are patterns over `lbits` (pat_a = the partner's
 * global-bit values moved onto the local bits, pat_b = a's).  q = 1,
 * pat_a = 1 << l, pat_b = 0 is dsv_exchange_halves.  complex64 moves whole
 * 16-byte units even when amplitude bit 0 is one of the local bits.
 * dsv_exchange_masked runs slice `part` of `nparts` on a's device (one
 * process per GPU: each partner runs one slice over a peer mapping). */
int dsv_exchange_masked(dsv_state* a, dsv_state* b, const int32_t* lbits, int q, uint64_t pat_a, uint64_t pat_b,
                        int part, int nparts);
/* One process driving both devices: half of the work on a's device and
 * stream, half on b's, both streams joined before and after (stream-ordered,
 * no host synchronisation; peer access enabled on first use). */
int dsv_exchange_pair(dsv_state* a, dsv_state* b, const int32_t* lbits, int q, uint64_t pat_a, uint64_t pat_b);
/* make `waiter`'s stream wait for everything queued so far on `other`'s */
int dsv_stream_join(dsv_state* waiter, dsv_state* other);

/* ---- sharded reductions (one segment per device, all devices at once) ---- */
/* The reduction of each segment is queued on its own stream, then all are
 * collected: out[i * per + j] = value j of segment i (per = 1 for norm2,
 * 2^k for marginals, 2 (re, im) for Pauli strings).  The caller combines the
 * per-segment values in a fixed order (deterministic; the reference's
 * SegmentedStateVector has no reductions of its own, BASELINE config 5). */
int dsv_group_norm2(dsv_state** s, int count, double* out);
int dsv_group_marginal_probs(dsv_state** s, int count, const int32_t* bits, int k, double* out);
int dsv_group_expect_pauli(dsv_state** s, int count, const int32_t* bits, const char* paulis, int m, double* out);

/* multi-process peers over NVLink: CUDA IPC handle of a segment (64 bytes) */
int dsv_ipc_handle(dsv_state* s, void* out64);
/* map a peer segment of the same nbits/dtype into this process as a state
 * handle owned by device `device` (the mapping is closed on destroy) */
int dsv_peer_open(int device, int nbits, int dtype, const void* handle64, dsv_state** out);

/* ---- CUDA graphs: record the device work of a gate sequence, replay it ---- */
/* Between dsv_capture_begin and dsv_capture_end the gate entry points of `s`
 * (apply_matrix / genperm / matrix_phased / pauli rotation and product /
 * swap_index_bits / set_basis / set_zero / scale) are recorded on the state's
 * stream instead of executed; per-gate tables are baked into buffers owned by
 * the graph.  Reductions, host transfers and exchanges return DSV_EINVAL while
 * capturing.  dsv_graph_launch replays the recorded work on the same state
 * (one launch for the whole sequence: the small-state circuits the host's
 * per-gate call overhead dominates). */
typedef struct dsv_graph dsv_graph;
int dsv_capture_begin(dsv_state* s);
int dsv_capture_end(dsv_state* s, dsv_graph** out);
int dsv_graph_launch(dsv_graph* g, dsv_state* s);
int dsv_graph_destroy(dsv_graph* g);

/* ---- instrumentation (bench.py) ----------------------------------------- */
/* When enabled, every kernel launched on `s` is bracketed by CUDA events on
 * the state's stream and tagged with its kernel class and algorithmic bytes
 * (SURVEY.md section 8(d)).  dsv_prof_read synchronises and aggregates:
 * for class c in [0, DSV_PROF_NCLASS): count[c], ms[c], bytes[c]. */
#define DSV_PROF_NCLASS 24
int dsv_prof_enable(dsv_state* s, int on);
int dsv_prof_reset(dsv_state* s);
int dsv_prof_read(dsv_state* s, uint64_t* count, double* ms, double* bytes);
const char* dsv_prof_class_name(int c);
/* events on the state's stream for whole-region timing */
int dsv_event_record(dsv_state* s, int slot);
int dsv_event_elapsed(dsv_state* s, int slot_a, int slot_b, float* ms);

#ifdef __cplusplus
}
#endif
#endif /* DSV_H */
