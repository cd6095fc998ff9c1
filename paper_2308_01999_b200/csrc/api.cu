// api.cu — the C ABI (include/dsv.h): state handles, argument validation,
// gate canonicalisation, kernel dispatch, instrumentation.
//
// Host-side responsibilities that the reference performs with NumPy index
// gymnastics (statevec.py:26-60) are done here once per gate in O(2^k):
//   * targets are sorted and the matrix / permutation re-indexed to the
//     sorted order, so kernels see canonical geometry;
//   * the control subcube + target positions become a Geom (hole insertion
//     masks) and 2^k member offsets;
//   * the access mode is chosen: complex64 with index bit 0 free runs on
//     128-bit float4 units holding two amplitudes.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/dsv.h"
#include "common.cuh"
#include "launch.h"

using namespace dsv;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
// The shared-memory tile path for low-target dense gates is opt-in
// (DSV_ENABLE_TILE=1): the sweep shows the register path ahead at every
// low-target position so far (profiles/sweep_r1_tile_ab.json).
const bool g_disable_tile = [] {
  const char* e = std::getenv("DSV_ENABLE_TILE");
  return !(e && e[0] == '1');
}();

// Tensor-core path for k = 4, 5 complex64 dense / phased windows (tc.cu).
// DSV_TC=0 disables it (A/B runs against the CUDA-core kernels).
bool g_tc_env = [] {
  const char* e = std::getenv("DSV_TC");
  return !(e && e[0] == '0');
}();

// 8-bit integer-digit tensor-core kernel for k = 4, 5 (tc8.cu); DSV_TC8=0 selects
// the bf16-limb kernel (tc.cu) instead.
bool g_tc8_env = [] {
  const char* e = std::getenv("DSV_TC8");
  return !(e && e[0] == '0');
}();

// Warp-specialised pipeline for the int8-digit kernel (tc8.cu k_dense_tc8ws);
// DSV_TC8WS=0 selects the two-group kernel.
bool g_tc8ws_env = [] {
  const char* e = std::getenv("DSV_TC8WS");
  return !(e && e[0] == '0');
}();
bool g_tc8ws_all = false;  // A/B: the warp-specialised pipeline for every plain tc8 window
bool g_tc8ws_row2 = true;

// complex128 k = 5 windows on the tensor cores through 8-bit digits at
// fp64-level accuracy (tc8d.cu); DSV_TC8D=0 keeps the FP64 CUDA-core kernels.
bool g_tc8d_env = [] {
  const char* e = std::getenv("DSV_TC8D");
  return !(e && e[0] == '0');
}();
bool g_tc8d512 = true;      // tc8d.cu: 512-thread layout (4 parts per row), else 256
bool g_tc8_pair01 = true;   // tc8 windows with targets on index bits 0 and 1 (member-pair mode 3)
// tc8 two-group kernel, plain row-pair windows: pair-swapped 16-byte stores
// (lane shuffles) instead of 8-byte row stores.  2 % faster on sparse data
// (QFT's first window on |0>), 8-12 % slower on a dense random state (QV /
// random circuits: (3,9,17,22,30) 27.0 -> 23.7 ms with 8-byte stores,
// tools/_st8_probe.py): off by default.  (The warp-specialised kernel keeps
// the pair-swapped stores: there they win on dense states, 31.5 -> 28.7 ms.)
bool g_tc8_pairswap = false;
bool g_tc4_all = false;  // A/B: every complex64 k = 4 dense gate on the tensor cores

// Launch-constant row phase vectors for windows whose row-varying phases sit
// on <= 3 tile-row bits (tc8.cu); DSV_ROWVEC=0 keeps the per-row sincos tree.
bool g_rowvec_env = [] {
  const char* e = std::getenv("DSV_ROWVEC");
  return !(e && e[0] == '0');
}();

// TMA tile loads for the int8-digit kernel's row-pair windows (tc8.cu kTcTma);
// DSV_TMA=0 keeps the per-thread cp.async copies.
bool g_tma_env = [] {
  const char* e = std::getenv("DSV_TMA");
  return !(e && e[0] == '0');
}();

// Lane-split kernel for k <= 3 complex64 windows on the lowest k bits (low.cu).
// DSV_LOW=0 disables it.
bool g_low_env = [] {
  const char* e = std::getenv("DSV_LOW");
  return !(e && e[0] == '0');
}();

// Warp-transposed phased k = 3 low-window kernel (low.cu k_dense_lowt); DSV_LOWT=0 disables.
bool g_lowt_env = [] {
  const char* e = std::getenv("DSV_LOWT");
  return !(e && e[0] == '0');
}();

// 64-byte-block kernel for complex64 dense gates inside bits 0..2 (perm.cu); DSV_DBLK8=0 disables.
bool g_dblk8_env = [] {
  const char* e = std::getenv("DSV_DBLK8");
  return !(e && e[0] == '0');
}();

// 64-byte-block kernel for complex64 permutations inside bits 0..2 (perm.cu); DSV_BLK8=0 disables.
bool g_blk8_env = [] {
  const char* e = std::getenv("DSV_BLK8");
  return !(e && e[0] == '0');
}();

// Warp-transpose kernel for dense gates inside the lowest 6 bits (wt.cu); DSV_WT=0 disables.
bool g_wt_env = [] {
  const char* e = std::getenv("DSV_WT");
  return !(e && e[0] == '0');
}();

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    return fail(DSV_ENOMEM, "%s: out of device memory (%s)", what, cudaGetErrorString(e));
  return fail(DSV_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(expr)                                         \
  do {                                                   \
    cudaError_t e_ = (expr);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr);  \
  } while (0)

#define CKL(expr, n)                                     \
  do {                                                   \
    cudaError_t e_ = (expr);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr);  \
    g_launches += (n);                                   \
  } while (0)

// NVTX ranges around the C-ABI entry points (names = the entry point), so an
// nsys / ncu --nvtx timeline lines kernels up with the calls that issued them.
// Off unless DSV_NVTX=1 (the push/pop pair is cheap, but not free per gate).
const bool g_nvtx_env = [] {
  const char* e = std::getenv("DSV_NVTX");
  return e && e[0] == '1';
}();
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name) : on(g_nvtx_env) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};
#define DSV_NVTX_RANGE() NvtxRange nvtx_range_(__func__)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

enum ProfClass {
  PC_DENSE = 0, PC_DENSE_GENERIC, PC_PERM, PC_PERM_GENERIC, PC_SWAP, PC_REDUCE,
  PC_EXPECT, PC_PAULI, PC_COLLAPSE, PC_EXCHANGE, PC_ACCESS, PC_SAMPLE,
  PC_DENSE_PHASED, PC_DIAG, PC_DENSE_TILE, PC_DENSE_TC, PC_DENSE_LOW, PC_DENSE_WT
};
const char* kProfNames[DSV_PROF_NCLASS] = {
    "dense", "dense_generic", "genperm", "genperm_generic", "swap_bits", "reduce",
    "expect", "pauli", "collapse", "exchange", "access", "sample",
    "dense_phased", "diag", "dense_tile", "dense_tc", "dense_low", "dense_wt"};

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double bytes;
};

}  // namespace

struct dsv_state {
  int device = 0;
  int nbits = 0;
  int dtype = 0;
  void* d = nullptr;
  bool owned = true;
  bool ipc = false;
  bool exported = false;  // an IPC handle was handed out: never recycle the allocation
  cudaStream_t stream = nullptr;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* gdata = nullptr;  // per-gate tables (stream-ordered reuse)
  size_t gdata_bytes = 0;
  bool prof_on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t uev[16] = {};
  // CUDA-graph capture (dsv_capture_begin/end): per-gate tables go to
  // buffers owned by the graph, filled at capture time
  bool capturing = false;
  std::vector<void*> cap_bufs;
  void* keep_gdata = nullptr;
  size_t keep_gdata_bytes = 0;
  void* keep_scratch = nullptr;
  size_t keep_scratch_bytes = 0;
  // deferred reductions (dsv_group_*): results land in pinned host memory and
  // the call returns before the GPU finishes
  bool defer = false;
  double* pinned = nullptr;
  size_t pinned_n = 0;
  size_t pending_n = 0;
};

namespace {

size_t amp_bytes(int dtype) { return dtype == DSV_C128 ? 16 : 8; }
uint64_t namps(const dsv_state* s) { return 1ull << s->nbits; }

// while capturing a graph every table gets its own buffer (the graph replays
// them later; the stream-ordered reuse of one buffer would alias them)
int capture_buffer(dsv_state* s, size_t bytes, void** out, size_t* out_bytes) {
  const size_t want = std::max<size_t>(bytes, 256);
  void* p = nullptr;
  CK(cudaMalloc(&p, want));
  s->cap_bufs.push_back(p);
  *out = p;
  *out_bytes = want;
  return DSV_OK;
}

int ensure_scratch(dsv_state* s, size_t bytes) {
  if (s->capturing) return capture_buffer(s, bytes, &s->scratch, &s->scratch_bytes);
  if (s->scratch_bytes >= bytes) return DSV_OK;
  if (s->scratch) {
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaFree(s->scratch));
    s->scratch = nullptr;
    s->scratch_bytes = 0;
  }
  size_t want = std::max<size_t>(bytes, size_t(1) << 20);
  CK(cudaMalloc(&s->scratch, want));
  s->scratch_bytes = want;
  return DSV_OK;
}

int ensure_gdata(dsv_state* s, size_t bytes) {
  if (s->capturing) return capture_buffer(s, bytes, &s->gdata, &s->gdata_bytes);
  if (s->gdata_bytes >= bytes) return DSV_OK;
  if (s->gdata) {
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaFree(s->gdata));
    s->gdata = nullptr;
    s->gdata_bytes = 0;
  }
  size_t want = std::max<size_t>(bytes, size_t(64) << 10);
  CK(cudaMalloc(&s->gdata, want));
  s->gdata_bytes = want;
  return DSV_OK;
}

// per-gate table upload: stream-ordered normally; baked synchronously into the
// graph-owned buffer while capturing (a captured memcpy would read the host
// temporary again at every replay)
cudaError_t h2d(dsv_state* s, void* dst, const void* src, size_t bytes) {
  if (s->capturing) return cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s->stream);
}

int no_capture(const dsv_state* s, const char* what) {
  if (s && s->capturing) return fail(DSV_EINVAL, "%s is not allowed while a graph is being captured", what);
  return DSV_OK;
}

cudaEvent_t pool_event(dsv_state* s) {
  if (!s->ev_pool.empty()) {
    cudaEvent_t e = s->ev_pool.back();
    s->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct ProfTok {
  cudaEvent_t a = nullptr;
};

ProfTok prof_start(dsv_state* s) {
  ProfTok t;
  if (s->prof_on && !s->capturing) {
    t.a = pool_event(s);
    cudaEventRecord(t.a, s->stream);
  }
  return t;
}

void prof_stop(dsv_state* s, ProfTok t, int cls, double bytes) {
  if (!s->prof_on || !t.a || s->capturing) return;
  cudaEvent_t b = pool_event(s);
  cudaEventRecord(b, s->stream);
  s->recs.push_back(ProfRec{cls, t.a, b, bytes});
}

int check_state(const dsv_state* s) {
  if (!s) return fail(DSV_EINVAL, "null state");
  return DSV_OK;
}

// Geometry over a unit index space of `ubits` bits with sorted holes.
int make_geom(int ubits, const std::vector<int>& holes_sorted, uint64_t set_mask, Geom* g) {
  const int H = int(holes_sorted.size());
  if (H > ubits) return fail(DSV_EINVAL, "more hole bits (%d) than index bits (%d)", H, ubits);
  if (H + 1 > DSV_MAX_GEOM_SEGS) return fail(DSV_EUNSUPPORTED, "too many hole bits");
  std::memset(g, 0, sizeof(Geom));
  g->nwork = 1ull << (ubits - H);
  g->set_mask = set_mask;
  g->nseg = 0;
  for (int i = 0; i <= H; ++i) {
    const int lo = i == 0 ? 0 : holes_sorted[i - 1] + 1;
    const int hi = i == H ? 64 : holes_sorted[i];
    uint64_t m = 0;
    for (int b = lo; b < hi; ++b) m |= 1ull << b;
    if (m == 0) continue;  // adjacent holes: empty run
    g->seg[g->nseg] = m;
    g->shift[g->nseg] = uint8_t(i);
    ++g->nseg;
  }
  return DSV_OK;
}

struct GateGeom {
  int k = 0, nctrl = 0;
  std::vector<int> tsorted;  // sorted targets (amp bits)
  std::vector<int> order;    // order[m'] = original target position of sorted m'
  std::vector<int> holes;    // sorted targets + control bits (amp bits)
  uint64_t set_mask = 0;     // amp space
};

int validate_gate(const dsv_state* s, const int32_t* targets, int k, const int32_t* cb,
                  const int32_t* cv, int nctrl, GateGeom* gg) {
  if (k < 0 || k > DSV_MAX_TARGETS)
    return fail(DSV_EINVAL, "gate arity %d outside [0, %d]", k, DSV_MAX_TARGETS);
  if (nctrl < 0) return fail(DSV_EINVAL, "negative control count");
  if (k > 0 && !targets) return fail(DSV_EINVAL, "null targets");
  if (nctrl > 0 && (!cb || !cv)) return fail(DSV_EINVAL, "null controls");
  uint64_t seen = 0;
  for (int m = 0; m < k; ++m) {
    const int t = targets[m];
    if (t < 0 || t >= s->nbits) return fail(DSV_EINVAL, "target bit %d out of range [0, %d)", t, s->nbits);
    if (seen >> t & 1) return fail(DSV_EINVAL, "duplicate bit %d", t);
    seen |= 1ull << t;
  }
  gg->set_mask = 0;
  for (int c = 0; c < nctrl; ++c) {
    const int b = cb[c];
    if (b < 0 || b >= s->nbits) return fail(DSV_EINVAL, "control bit %d out of range [0, %d)", b, s->nbits);
    if (seen >> b & 1) return fail(DSV_EINVAL, "targets/controls overlap at bit %d", b);
    if (cv[c] != 0 && cv[c] != 1) return fail(DSV_EINVAL, "control value %d not in {0,1}", cv[c]);
    seen |= 1ull << b;
    if (cv[c]) gg->set_mask |= 1ull << b;
  }
  gg->k = k;
  gg->nctrl = nctrl;
  gg->order.resize(k);
  for (int m = 0; m < k; ++m) gg->order[m] = m;
  std::sort(gg->order.begin(), gg->order.end(),
            [&](int x, int y) { return targets[x] < targets[y]; });
  gg->tsorted.resize(k);
  for (int m = 0; m < k; ++m) gg->tsorted[m] = targets[gg->order[m]];
  gg->holes.clear();
  for (int b = 0; b < 64; ++b)
    if (seen >> b & 1) gg->holes.push_back(b);
  return DSV_OK;
}

// index j' in sorted-target order -> index j in caller order
inline uint64_t old_index(const GateGeom& gg, uint64_t jn) {
  uint64_t j = 0;
  for (int m = 0; m < gg.k; ++m) j |= ((jn >> m) & 1ull) << gg.order[m];
  return j;
}
inline uint64_t new_index(const GateGeom& gg, uint64_t j) {
  uint64_t jn = 0;
  for (int m = 0; m < gg.k; ++m) jn |= ((j >> gg.order[m]) & 1ull) << m;
  return jn;
}

// unit-space view of a gate: VEC2 when complex64 and index bit 0 is not a hole
struct UnitView {
  int mode;
  int ubits;
  int shift;
  Geom g;
  std::vector<uint64_t> offs;  // 2^k member offsets (units)
};

int unit_view(const dsv_state* s, const GateGeom& gg, bool allow_vec2, UnitView* uv) {
  const bool bit0_hole = !gg.holes.empty() && gg.holes[0] == 0;
  uv->mode = (s->dtype == DSV_C64 && allow_vec2 && !bit0_hole && s->nbits >= 1) ? MODE_VEC2 : MODE_SCALAR;
  uv->shift = uv->mode == MODE_VEC2 ? 1 : 0;
  uv->ubits = s->nbits - uv->shift;
  std::vector<int> h(gg.holes);
  for (int& x : h) x -= uv->shift;
  int rc = make_geom(uv->ubits, h, gg.set_mask >> uv->shift, &uv->g);
  if (rc) return rc;
  const uint64_t D = 1ull << gg.k;
  uv->offs.assign(D, 0);
  for (uint64_t j = 0; j < D; ++j) {
    uint64_t o = 0;
    for (int m = 0; m < gg.k; ++m) o |= ((j >> m) & 1ull) << (gg.tsorted[m] - uv->shift);
    uv->offs[j] = o;
  }
  return DSV_OK;
}

template <typename R>
void canon_matrix(const GateGeom& gg, const void* m_in, std::vector<cplx<R>>& out) {
  const uint64_t D = 1ull << gg.k;
  const cplx<R>* m = static_cast<const cplx<R>*>(m_in);
  std::vector<uint64_t> old(D);
  for (uint64_t j = 0; j < D; ++j) old[j] = old_index(gg, j);
  out.resize(D * D);
  for (uint64_t r = 0; r < D; ++r)
    for (uint64_t c = 0; c < D; ++c) out[r * D + c] = m[old[r] * D + old[c]];
}

// sm_100-class device (tcgen05 available)?
bool device_has_tcgen05(int dev) {
  static int cache[64] = {0};  // 0 unknown, 1 yes, 2 no
  if (dev < 0 || dev >= 64) return false;
  if (!cache[dev]) {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cache[dev] = major == 10 ? 1 : 2;
  }
  return cache[dev] == 1;
}

struct PhaseTerm {
  int slot;  // sorted target position m (< k), or k for an outside-only term
  int bit;   // amplitude index bit (outside the targets)
  double th;
};

// Can the tensor-core kernel take this gate?  complex64, k in {4, 5}, whole
// 128-group tiles.  Index bit 0 free selects 16-byte row-pair copies (PAIR),
// else each thread moves its own row 8 bytes per member.
// 2: targets exactly bits 0..k-1 and no control below bit k + 7 (tiles of 128
// groups are contiguous); 1: index bit 0 free; 0: otherwise
int tc_mode(const GateGeom& gg) {
  bool low = true;
  for (int m = 0; m < gg.k; ++m) low = low && gg.tsorted[m] == m;
  if (low) {
    for (int b : gg.holes)
      if (b >= gg.k && b < gg.k + 7) low = false;
    if (low) return 2;
  }
  return gg.holes[0] != 0 ? 1 : 0;
}

bool tc_eligible(const dsv_state* s, const GateGeom& gg) {
  if (!g_tc_env || s->dtype != DSV_C64) return false;
  if (gg.k < 4 || gg.k > 6) return false;
  // k = 6 with index bits 0 and 1 both holes: tc68's per-row 8-byte copies
  // waste half of each sector, but the alternative is the generic CUDA-core
  // kernel (QV-33 k = 6 windows: ~420 ms each there), so they stay here
  // rows are the lowest free bits: with bits 0 and 1 both holes, consecutive
  // rows sit >= 32 bytes apart and the per-row 8-byte copies waste sectors —
  // unless the targets are exactly bits 0..k-1 (contiguous tiles, mode 2)
  // (tc8, k <= 5: index bit 0 the lowest target moves member pairs as 16-byte
  // units (mode 3), so bits 0 and 1 both targets are fine there: QV-33 k = 5
  // windows on (0, 1, ..) 88 -> ~25 ms)
  if (gg.holes.size() >= 2 && gg.holes[0] == 0 && gg.holes[1] == 1 && tc_mode(gg) != 2 && gg.k <= 5 &&
      !(g_tc8_env && gg.tsorted[0] == 0 && gg.tsorted[1] == 1 && g_tc8_pair01))
    return false;
  const int free_bits = s->nbits - gg.k - gg.nctrl;
  if (free_bits < 7) return false;
  return device_has_tcgen05(s->device);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeTiledFn(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// kTcTma eligibility + tensor map: complex64 state, no controls, index bit 0
// free, rows = the 7 lowest free bits.  Index bits are labelled row / member
// / tile and cut into runs of equal labels; the map's dimensions are the runs
// (at most 5) ordered rows first, then members, then tile runs, so the box
// (all rows x all members x one tile) lands as [member][row] in shared
// memory — the layout the kernel's converters read.  Returns false (and the
// caller keeps cp.async) when the layout needs more than 5 runs or the driver
// rejects the map.
bool build_tile_tmap(const dsv_state* s, const GateGeom& gg, TcDesc* d) {
  if (!g_tma_env || gg.nctrl != 0 || gg.k > 5 || s->dtype != DSV_C64) return false;
  const int n = s->nbits;
  std::vector<char> lab(n, 'T');
  for (int m = 0; m < gg.k; ++m) lab[gg.tsorted[m]] = 'M';
  if (lab[0] != 'T') return false;  // bit 0 must be a row bit
  for (int b = 0, rows = 0; b < n && rows < 7; ++b)
    if (lab[b] == 'T') {
      lab[b] = 'R';
      ++rows;
    }
  struct Run { char l; int start, len; };
  std::vector<Run> runs;
  for (int b = 0; b < n; ++b) {
    if (!runs.empty() && runs.back().l == lab[b] && runs.back().start + runs.back().len == b) ++runs.back().len;
    else runs.push_back({lab[b], b, 1});
  }
  if (runs.size() > 5) return false;
  std::vector<Run> order;
  for (char l : {'R', 'M', 'T'})
    for (const Run& r : runs)
      if (r.l == l) order.push_back(r);
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5];
  int consumed = 0;  // tile runs appear in ascending bit order: tile index bits map low -> high
  for (int q = 0; q < 5; ++q) {
    estr[q] = 1;
    d->tma_shift[q] = 0;
    d->tma_mask[q] = 0;
    if (q < int(order.size())) {
      dims[q] = cuuint64_t(1) << order[q].len;
      box[q] = order[q].l == 'T' ? 1u : cuuint32_t(1) << order[q].len;
      if (q) strides[q - 1] = (cuuint64_t(1) << order[q].start) * 8;
      if (order[q].l == 'T') {
        if (order[q].len > 31) return false;
        d->tma_shift[q] = consumed;
        d->tma_mask[q] = (uint32_t(1) << order[q].len) - 1u;
        consumed += order[q].len;
      }
    } else {  // padding dimension of extent 1
      dims[q] = 1;
      box[q] = 1;
      strides[q - 1] = (cuuint64_t(1) << n) * 8;
    }
  }
  if (order[0].l != 'R' || order[0].start != 0) return false;
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return false;
  const CUresult r = fn(&d->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, s->d, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Unit factors exp(i angle) per (index-byte chunk, byte value, slot) for a
// phased window's terms (slots 0..k-1: member bits, k: every member), in the
// state's precision: [nchunk][256][k + 1] complex.  chunk_shift[c] = 8 * byte.
void unit_factor_tables(const std::vector<PhaseTerm>& terms, int k, bool c128, int* nchunk, int chunk_shift[8],
                        std::vector<unsigned char>& raw) {
  int chunk_of_byte[8];
  for (int c = 0; c < 8; ++c) chunk_of_byte[c] = -1;
  *nchunk = 0;
  for (const PhaseTerm& t : terms) {
    const int c = t.bit / 8;
    if (chunk_of_byte[c] < 0) {
      chunk_of_byte[c] = *nchunk;
      chunk_shift[(*nchunk)++] = 8 * c;
    }
  }
  const int S = k + 1;
  const size_t nt = size_t(std::max(*nchunk, 1)) * 256 * S;
  std::vector<double> tab(nt, 0.0);
  for (const PhaseTerm& t : terms) {
    const int ci = chunk_of_byte[t.bit / 8];
    const int bb = t.bit % 8;
    for (int v = 0; v < 256; ++v)
      if ((v >> bb) & 1) tab[(size_t(ci) * 256 + v) * S + t.slot] += t.th;
  }
  const size_t es = c128 ? 16 : 8;
  raw.assign(nt * es, 0);
  for (size_t i = 0; i < nt; ++i) {
    const double c = std::cos(tab[i]), sn = std::sin(tab[i]);
    if (c128) {
      reinterpret_cast<double*>(raw.data())[2 * i] = c;
      reinterpret_cast<double*>(raw.data())[2 * i + 1] = sn;
    } else {
      reinterpret_cast<float*>(raw.data())[2 * i] = float(c);
      reinterpret_cast<float*>(raw.data())[2 * i + 1] = float(sn);
    }
  }
}

// every entry of the k-qubit matrix (state dtype) finite?
bool matrix_finite(const dsv_state* s, const void* matrix, int k) {
  const size_t n = size_t(2) << (2 * k);  // re + im
  if (s->dtype == DSV_C128) {
    const double* m = static_cast<const double*>(matrix);
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(m[i])) return false;
  } else {
    const float* m = static_cast<const float*>(matrix);
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(m[i])) return false;
  }
  return true;
}

// complex128 k = 5 dense window on the tensor cores (tc8d.cu)
bool tc8d_eligible(const dsv_state* s, const GateGeom& gg) {
  if (!g_tc_env || !g_tc8d_env || s->dtype != DSV_C128 || gg.k != 5) return false;
  if (s->nbits - gg.k - gg.nctrl < 7) return false;
  return device_has_tcgen05(s->device);
}

// Gate digits: the real embedding E (n = 2i + out re/im, kk = 2j + in re/im)
// as X = rint(E 2^(51 - e_b)), |X| <= 2^51, and X + 0x0080808080808080 split
// into balanced base-256 digits b0 (2^48, |b0| <= 8) .. b6; row n of the
// 256 x 128 B table holds [b_(n/64) | b_(4 + n/64)] of output real n % 64.
int apply_tc8d(dsv_state* s, const GateGeom& gg, const void* matrix, const std::vector<PhaseTerm>& terms,
               int prof_class, double bytes) {
  constexpr int D = 32;
  UnitView uv;
  if (int rc = unit_view(s, gg, false, &uv)) return rc;
  TcDesc d;
  std::memset(&d, 0, sizeof d);
  d.g = uv.g;
  for (int j = 0; j < D; ++j) d.offs[j] = uv.offs[j];
  d.tshift = gg.tsorted[0];
  for (int m = 1; m < gg.k; ++m)
    if (gg.tsorted[m] != gg.tsorted[0] + m) d.tshift = -1;
  std::vector<cplx<double>> m;
  canon_matrix<double>(gg, matrix, m);
  double bmax = 0.0;
  for (const auto& z : m) bmax = std::max(bmax, std::max(std::fabs(z.x), std::fabs(z.y)));
  if (!std::isfinite(bmax)) return fail(DSV_EINVAL, "matrix has non-finite entries");
  int e_b = 0;
  if (bmax > 0.0) std::frexp(bmax, &e_b);  // bmax in [2^(e_b-1), 2^e_b)
  d.e_b = e_b;
  d.ws = g_tc8d512 ? 1 : 0;  // 512-thread layout (4 parts per row); dsv_config_set("tc8d512", 0): 256
  constexpr uint64_t kOff = 0x0080808080808080ull;
  std::vector<unsigned char> host(256 * 128, 0);
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      const double re = m[size_t(i) * D + j].x, im = m[size_t(i) * D + j].y;
      const double e[2][2] = {{re, -im}, {im, re}};
      for (int oc = 0; oc < 2; ++oc)
        for (int ic = 0; ic < 2; ++ic) {
          const int n = 2 * i + oc, kk = 2 * j + ic;
          const int64_t x = int64_t(std::nearbyint(std::ldexp(e[oc][ic], 51 - e_b)));
          const uint64_t u = uint64_t(x) + kOff;
          for (int pl = 0; pl < 7; ++pl) {
            const unsigned char byte = static_cast<unsigned char>(((u >> (8 * (6 - pl))) & 255u) ^ 0x80u);
            const int row = (pl < 4 ? pl : pl - 4) * 64 + n;
            host[size_t(row) * 128 + (pl < 4 ? 0 : 64) + kk] = byte;
          }
        }
    }
  // phased windows (fold fuser): unit-factor tables after the gate digits
  std::vector<unsigned char> ftab;
  if (!terms.empty()) {
    unit_factor_tables(terms, gg.k, true, &d.nnib, d.nib_shift, ftab);
    host.insert(host.end(), ftab.begin(), ftab.end());
  }
  if (int rc = ensure_gdata(s, host.size())) return rc;
  CK(h2d(s, s->gdata, host.data(), host.size()));
  ProfTok t = prof_start(s);
  CKL(launch_dense_tc8d(d, s->gdata, static_cast<const unsigned char*>(s->gdata) + 256 * 128, s->d, s->stream), 1);
  prof_stop(s, t, prof_class, bytes);
  return DSV_OK;
}

// Dense (+ optional pre-phase) window on the tensor cores; caller holds the device guard.
int apply_tc(dsv_state* s, const GateGeom& gg, const void* matrix, const std::vector<PhaseTerm>& terms,
             int prof_class, double bytes) {
  const int k = gg.k;
  const int D = 1 << k, KK = 2 * D;
  UnitView uv;
  if (int rc = unit_view(s, gg, false, &uv)) return rc;
  TcDesc d;
  std::memset(&d, 0, sizeof d);
  d.g = uv.g;
  d.mode = tc_mode(gg);
  // tc8 (k <= 5): index bit 0 the lowest target -> member pairs move as 16-byte units
  if (d.mode == 0 && k <= 5 && gg.tsorted[0] == 0 && g_tc8_env) d.mode = 3;  // kTcRow2 (tcgen05.cuh)
  if ((d.mode == 0 || d.mode == 2) && k == 6 && gg.tsorted[0] == 0 && g_tc8_env) d.mode = 3;  // tc68.cu row2 (member pairs)
  for (int j = 0; j < D; ++j) d.offs[j] = uv.offs[j];
  d.tshift = gg.tsorted[0];
  for (int m = 1; m < k; ++m)
    if (gg.tsorted[m] != gg.tsorted[0] + m) d.tshift = -1;
  // tile rows = the lowest 7 free (non-hole) index bits
  uint64_t row_mask = 0;
  {
    uint64_t hole_mask = 0;
    for (int b : gg.holes) hole_mask |= 1ull << b;
    for (int b = 0, got = 0; b < s->nbits && got < 7; ++b)
      if (!(hole_mask >> b & 1)) {
        row_mask |= 1ull << b;
        ++got;
      }
  }
  std::vector<cplx<float>> m;
  canon_matrix<float>(gg, matrix, m);
  float bmax = 0.f;
  for (const auto& z : m) bmax = std::max(bmax, std::max(std::fabs(z.x), std::fabs(z.y)));
  int e_b = 0;
  if (bmax > 0.f) std::frexp(bmax, &e_b);  // bmax in [2^(e_b-1), 2^e_b)
  const bool use_tc8 = g_tc8_env && k <= 6 && e_b >= -20 && e_b <= 20;
  // Row-varying phases on at most 3 tile-row bits (e.g. QFT-33's window on
  // qubits 3..7, whose CP partners 0..2 are row bits): the row part of the
  // phase depends only on those bits, so it is 2^nrb launch-constant vectors
  // R_v[j] built here; the kernel multiplies them into the tile-uniform
  // vector once per tile (nrb x 32 complex products in one warp) and every
  // row then takes one complex product per member, as for tile-uniform
  // windows, instead of a per-row 6-sincos tree.
  std::vector<int> rb_bits;
  for (const PhaseTerm& t : terms)
    if ((row_mask >> t.bit & 1) && std::find(rb_bits.begin(), rb_bits.end(), t.bit) == rb_bits.end())
      rb_bits.push_back(t.bit);
  std::sort(rb_bits.begin(), rb_bits.end());
  const bool rowvec = use_tc8 && k <= 5 && !rb_bits.empty() && rb_bits.size() <= 3 && g_rowvec_env;
  auto in_rb = [&](int bit) { return rowvec && std::find(rb_bits.begin(), rb_bits.end(), bit) != rb_bits.end(); };
  // phase slots per index nibble: [nnib][16][8]; nibbles holding a term on a
  // row bit come first (d.nnib_row of them: the per-row lookups), the rest are
  // uniform over a tile (coop = no per-row nibble at all)
  int nib_of[16];
  for (int c = 0; c < 16; ++c) nib_of[c] = -1;
  uint32_t rowvar = 0, used = 0;
  for (const PhaseTerm& t : terms) {
    if (in_rb(t.bit)) continue;
    const int c = t.bit / 4;
    if (c >= 10) return fail(DSV_EUNSUPPORTED, "tensor-core phase table covers index bits < 40");
    used |= 1u << c;
    if (row_mask >> t.bit & 1) rowvar |= 1u << c;
  }
  for (int pass = 0; pass < 2; ++pass)
    for (int c = 0; c < 10; ++c)
      if ((used >> c & 1) && ((rowvar >> c & 1) == (pass == 0 ? 1u : 0u))) {
        nib_of[c] = d.nnib;
        d.nib_shift[d.nnib++] = 4 * c;
        if (pass == 0) ++d.nnib_row;
      }
  d.coop = d.nnib_row == 0 ? 1 : 0;
  std::vector<double> tab(size_t(d.nnib) * 16 * 8, 0.0);
  for (const PhaseTerm& t : terms) {
    if (in_rb(t.bit)) continue;
    const int ci = nib_of[t.bit / 4], bb = t.bit % 4;
    for (int v = 0; v < 16; ++v)
      if ((v >> bb) & 1) tab[(size_t(ci) * 16 + v) * 8 + t.slot] += t.th;
  }
  std::vector<float> rvec;  // [2^nrb][D] (cos, sin)
  if (rowvec) {
    d.nrb = int(rb_bits.size());
    for (int q = 0; q < d.nrb; ++q) d.rb_bit[q] = rb_bits[q];
    rvec.assign(size_t(2) * D << d.nrb, 0.f);
    for (int v = 0; v < (1 << d.nrb); ++v)
      for (int j = 0; j < D; ++j) {
        double ang = 0.0;
        for (const PhaseTerm& t : terms) {
          if (!in_rb(t.bit)) continue;
          const int q = int(std::find(rb_bits.begin(), rb_bits.end(), t.bit) - rb_bits.begin());
          if (!((v >> q) & 1)) continue;
          if (t.slot < k && !((j >> t.slot) & 1)) continue;
          ang += t.th;
        }
        rvec[(size_t(v) * D + j) * 2] = float(std::cos(ang));
        rvec[(size_t(v) * D + j) * 2 + 1] = float(std::sin(ang));
      }
  }
  if (use_tc8) {
    // 8-bit digits (tc8.cu): X = B 2^(23 - e_b) rounded, X + 0x8080 split into
    // balanced base-256 digits b2 (2^16), b1 (2^8), b0 in [-128, 127];
    // rows [b2 | b1 | b0] x (n = 2i + out re/im), 128 bytes of K = 2j + in re/im
    constexpr int64_t kLim = (int64_t(1) << 23) - 0x8080 - 1;
    std::vector<int64_t> X(size_t(KK) * KK);
    for (int tries = 0; tries < 2; ++tries) {
      int64_t xmax = 0;
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
          const float re = m[size_t(i) * D + j].x, im = m[size_t(i) * D + j].y;
          const float e[2][2] = {{re, -im}, {im, re}};
          for (int oc = 0; oc < 2; ++oc)
            for (int ic = 0; ic < 2; ++ic) {
              const int64_t x = int64_t(std::nearbyint(std::ldexp(double(e[oc][ic]), 23 - e_b)));
              X[size_t(2 * i + oc) * KK + (2 * j + ic)] = x;
              xmax = std::max(xmax, x < 0 ? -x : x);
            }
        }
      if (xmax <= kLim) break;
      ++e_b;  // the rounded maximum reached the digit range: one more bit of headroom
    }
    d.e_b = e_b;
    // warp-specialised pipeline only where it measured faster on the same box
    // (tools/_patt2.py, _ab_qft.py, _ab_qvwin.py at n = 33): plain windows
    // with index bit 0 the lowest target (member pairs as 16-byte units,
    // 0.87-0.89 -> 0.97 of the copy peak) or with the lowest target at bit 1
    // or 2 (QV windows 34.0 -> 31.1 ms and 28.3 -> 27.5 ms).  Elsewhere it is
    // a wash or up to 5 % slower (contiguous and phased windows, targets from
    // bit 3 up): DSV_TC8WS=0 disables it; dsv_config_set("tc8ws_all", 1)
    // forces it for A/B runs.
    d.pairswap = g_tc8_pairswap ? 1 : 0;
    const bool ws_layout = (d.mode == 3 && g_tc8ws_row2) || (d.mode == 1 && gg.tsorted[0] <= 2);
    d.ws = (g_tc8ws_env && terms.empty() && (ws_layout || g_tc8ws_all)) ? 1 : 0;
    // TMA tile loads where they measured faster than the per-thread cp.async
    // copies (tools/_ab_tma.py, same box, n = 33): windows whose 128 tile rows
    // are split around the targets (lowest target below bit 7, e.g. QFT-33's
    // window on qubits 3..7: 27.5 -> 27.1 ms).  Rows that are one contiguous
    // run (plain windows high up: 22.5 -> 24.4 ms) keep cp.async.
    // The box's innermost run is the rows below the lowest target: under
    // 64 bytes (lowest target bit 1 or 2) TMA moves 16-32-byte pieces and
    // was measured slower (QV windows with targets from bit 1: 31 -> 34.8
    // ms), so those keep cp.async with the row-pair mapping of tc8.cu.
    if (k <= 5 && d.mode == 1 && gg.tsorted[0] >= 3 && gg.tsorted[0] < 7 && build_tile_tmap(s, gg, &d))
      d.mode = 4;  // kTcTma
    std::vector<unsigned char> host8(size_t(3) * KK * 128, 0);
    for (int n = 0; n < KK; ++n)
      for (int kk = 0; kk < KK; ++kk) {
        const int64_t xp = X[size_t(n) * KK + kk] + 0x8080;
        const int dig[3] = {int(xp >> 16), int((xp >> 8) & 255) - 128, int(xp & 255) - 128};
        for (int l = 0; l < 3; ++l) host8[(size_t(l) * KK + n) * 128 + kk] = static_cast<unsigned char>(int8_t(dig[l]));
      }
    const size_t bbytes = (host8.size() + 255) / 256 * 256;
    const size_t tbytes = (tab.size() * sizeof(float) + 255) / 256 * 256;
    std::vector<unsigned char> host(bbytes + tbytes + rvec.size() * sizeof(float), 0);
    std::memcpy(host.data(), host8.data(), host8.size());
    for (size_t i = 0; i < tab.size(); ++i) {
      const float f = float(tab[i]);
      std::memcpy(host.data() + bbytes + i * 4, &f, 4);
    }
    if (!rvec.empty()) std::memcpy(host.data() + bbytes + tbytes, rvec.data(), rvec.size() * sizeof(float));
    if (int rc = ensure_gdata(s, host.size())) return rc;
    CK(h2d(s, s->gdata, host.data(), host.size()));
    const unsigned char* d_b = static_cast<const unsigned char*>(s->gdata);
    d.htab = reinterpret_cast<const float*>(host.data() + bbytes);
    d.d_rvec = rvec.empty() ? nullptr : d_b + bbytes + tbytes;
    ProfTok t = prof_start(s);
    if (k == 6)
      CKL(launch_dense_tc68(d, d_b, d_b + bbytes, s->d, s->stream), 1);
    else
      CKL(launch_dense_tc8(k, d, d_b, d_b + bbytes, s->d, s->stream), 1);
    prof_stop(s, t, prof_class, bytes);
    return DSV_OK;
  }
  // real embedding of the canonical matrix (n = 2i + out re/im, kk = 2j + in
  // re/im) as 2^(e_b - 8) (b0 + b1 / 2^8 + b2 / 2^16), exact bf16 limbs
  // [b0, b1, b2 / 2^8, b1 / 2^8][n][64] (tc.cu)
  const int KP = KK < 64 ? 64 : KK;  // whole 128-byte bf16 K blocks per B row
  const int nlimb = k == 6 ? 3 : 4;  // k = 6: b0, b1, b2 / 2^8 (a1 / 2^8 rides on the A side)
  d.e_b = e_b;
  const size_t limb_elems = size_t(KK) * KP;
  std::vector<uint16_t> limbs(size_t(nlimb) * limb_elems, 0);
  auto bf16_bits = [](float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    return uint16_t(u >> 16);  // exact: small integers times powers of two
  };
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      const float re = m[size_t(i) * D + j].x, im = m[size_t(i) * D + j].y;
      const float e[2][2] = {{re, -im}, {im, re}};  // [out re/im][in re/im]
      for (int oc = 0; oc < 2; ++oc)
        for (int ic = 0; ic < 2; ++ic) {
          // I = e 2^(24 - e_b), |I| < 2^24: exact for a float (no rounding)
          const double I = std::ldexp(double(e[oc][ic]), 24 - e_b);
          const double b0 = std::nearbyint(I / 65536.0);
          const double rem = I - b0 * 65536.0;
          const double b1 = std::nearbyint(rem / 256.0);
          const double b2 = rem - b1 * 256.0;
          const size_t at = size_t(2 * i + oc) * KP + (2 * j + ic);
          limbs[at] = bf16_bits(float(b0));
          limbs[limb_elems + at] = bf16_bits(float(b1));
          limbs[2 * limb_elems + at] = bf16_bits(float(b2 / 256.0));
          if (nlimb > 3) limbs[3 * limb_elems + at] = bf16_bits(float(b1 / 256.0));
        }
    }
  const size_t limb_bytes = (limbs.size() * 2 + 255) / 256 * 256;
  std::vector<unsigned char> host(limb_bytes + tab.size() * sizeof(float), 0);
  std::memcpy(host.data(), limbs.data(), limbs.size() * 2);
  for (size_t i = 0; i < tab.size(); ++i) {
    const float f = float(tab[i]);
    std::memcpy(host.data() + limb_bytes + i * 4, &f, 4);
  }
  if (int rc = ensure_gdata(s, host.size())) return rc;
  CK(h2d(s, s->gdata, host.data(), host.size()));
  const unsigned char* d_b = static_cast<const unsigned char*>(s->gdata);
  d.htab = reinterpret_cast<const float*>(host.data() + limb_bytes);
  ProfTok t = prof_start(s);
  if (k == 6)
    CKL(launch_dense_tc6(d, d_b, d_b + limb_bytes, s->d, s->stream), 1);
  else
    CKL(launch_dense_tc(k, d, d_b, d_b + limb_bytes, s->d, s->stream), 1);
  prof_stop(s, t, prof_class, bytes);
  return DSV_OK;
}

// complex64, 1 <= k <= 3, targets exactly bits 0..k-1, whole warps of lanes
bool low_eligible(const dsv_state* s, const GateGeom& gg) {
  if (!g_low_env || s->dtype != DSV_C64 || gg.k < 1 || gg.k > 3) return false;
  for (int m = 0; m < gg.k; ++m)
    if (gg.tsorted[m] != m) return false;
  // lane-items (groups x 2^(k-1)) fill whole 1024-item passes: no tail guards
  const int L = 1 << (gg.k - 1);
  const int free_bits = s->nbits - gg.k - gg.nctrl;
  return free_bits >= 0 && (std::ldexp(1.0, free_bits) * L) >= 1024.0;
}

// Low-target window (+ optional pre-phase); caller holds the device guard.
int apply_low(dsv_state* s, const GateGeom& gg, const void* matrix, const std::vector<PhaseTerm>& terms,
              int prof_class, double bytes) {
  const int k = gg.k;
  UnitView uv;
  if (int rc = unit_view(s, gg, false, &uv)) return rc;
  LowDesc d;
  std::memset(&d, 0, sizeof d);
  d.g = uv.g;
  d.plain = gg.nctrl == 0;
  // phase slots by index byte: [8][256][4] (bytes without terms stay zero)
  uint32_t used = 0;
  for (const PhaseTerm& t : terms) used |= 1u << (t.bit / 8);
  for (int c = 0; c < 8; ++c)
    if (used >> c & 1) d.chunk_shift[d.nchunk++] = 8 * c;
  if (!terms.empty()) {
    std::vector<double> tab(size_t(8) * 256 * 4, 0.0);
    for (const PhaseTerm& t : terms) {
      const int c = t.bit / 8, bb = t.bit % 8;
      for (int v = 0; v < 256; ++v)
        if ((v >> bb) & 1) tab[(size_t(c) * 256 + v) * 4 + t.slot] += t.th;
    }
    std::vector<float> host(tab.size());
    for (size_t i = 0; i < tab.size(); ++i) host[i] = float(tab[i]);
    if (int rc = ensure_gdata(s, host.size() * sizeof(float))) return rc;
    CK(h2d(s, s->gdata, host.data(), host.size() * sizeof(float)));
  }
  std::vector<cplx<float>> m;
  canon_matrix<float>(gg, matrix, m);
  ProfTok t = prof_start(s);
  if (g_lowt_env && d.plain && s->nbits >= 12)
    CKL(launch_dense_lowt(k, d, uint64_t(1) << s->nbits, m.data(), s->gdata, s->d, s->stream), 1);
  else
    CKL(launch_dense_low(k, d, m.data(), s->gdata, s->d, s->stream), 1);
  prof_stop(s, t, prof_class, bytes);
  return DSV_OK;
}

int sync_streams(dsv_state* waiter, dsv_state* other) {
  if (waiter->stream == other->stream) return DSV_OK;
  cudaEvent_t e;
  {
    DeviceGuard g(other->device);
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, other->stream));
  }
  CK(cudaStreamWaitEvent(waiter->stream, e, 0));
  cudaEventDestroy(e);
  return DSV_OK;
}

std::mutex g_peer_mu;
bool g_peer_enabled[64][64];

int enable_peer(int from, int to) {
  if (from == to) return DSV_OK;
  std::lock_guard<std::mutex> lk(g_peer_mu);
  if (g_peer_enabled[from][to]) return DSV_OK;
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, from, to));
  if (!can) return fail(DSV_EUNSUPPORTED, "device %d cannot access peer %d", from, to);
  DeviceGuard g(from);
  cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  cudaGetLastError();
  g_peer_enabled[from][to] = true;
  return DSV_OK;
}

// Small pinned host buffers for deferred reductions (dsv_group_*), kept in a
// process-wide free list: cudaMallocHost / cudaFreeHost cost milliseconds and
// synchronise the device, and a sharded state is rebuilt per circuit.
std::mutex g_pinned_mu;
std::vector<std::pair<double*, size_t>> g_pinned_free;

bool pinned_take(size_t n, double** out, size_t* out_n) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  for (size_t i = 0; i < g_pinned_free.size(); ++i)
    if (g_pinned_free[i].second >= n) {
      *out = g_pinned_free[i].first;
      *out_n = g_pinned_free[i].second;
      g_pinned_free.erase(g_pinned_free.begin() + long(i));
      return true;
    }
  return false;
}

void pinned_put(double* p, size_t n) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  if (g_pinned_free.size() < 64) g_pinned_free.push_back({p, n});
  else cudaFreeHost(p);
}

// reduce partials already on device -> host doubles
int finish_reduce(dsv_state* s, uint64_t nbins, uint64_t nchunks, int ncomp, double* d_partial,
                  double* d_out, double* host_out) {
  CKL(launch_final_sum(nbins, nchunks, ncomp, d_partial, d_out, s->stream), 1);
  if (s->defer) {  // dsv_group_*: copy into pinned memory, collect later
    const size_t n = size_t(nbins) * ncomp;
    if (s->pinned_n < n) {
      if (s->pinned) {
        CK(cudaStreamSynchronize(s->stream));
        pinned_put(s->pinned, s->pinned_n);
        s->pinned = nullptr;
        s->pinned_n = 0;
      }
      const size_t want = std::max<size_t>(n, 512);
      if (!pinned_take(want, &s->pinned, &s->pinned_n)) {
        CK(cudaMallocHost(&s->pinned, sizeof(double) * want));
        s->pinned_n = want;
      }
    }
    CK(cudaMemcpyAsync(s->pinned, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
    s->pending_n = n;
    return DSV_OK;
  }
  CK(cudaMemcpyAsync(host_out, d_out, sizeof(double) * nbins * ncomp, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return DSV_OK;
}

struct PauliMasks {
  uint64_t x = 0, yz = 0;
  int ny = 0, h = -1;
};

int parse_pauli(const dsv_state* s, const int32_t* bits, const char* paulis, int m, PauliMasks* pm) {
  if (m < 0) return fail(DSV_EINVAL, "negative Pauli length");
  uint64_t seen = 0;
  for (int i = 0; i < m; ++i) {
    const int b = bits[i];
    if (b < 0 || b >= s->nbits) return fail(DSV_EINVAL, "Pauli bit %d out of range [0, %d)", b, s->nbits);
    if (seen >> b & 1) return fail(DSV_EINVAL, "duplicate qubit in Pauli string: bit %d", b);
    seen |= 1ull << b;
    switch (paulis[i]) {
      case 'I': case 'i': break;
      case 'X': case 'x': pm->x |= 1ull << b; break;
      case 'Y': case 'y': pm->x |= 1ull << b; pm->yz |= 1ull << b; pm->ny++; break;
      case 'Z': case 'z': pm->yz |= 1ull << b; break;
      default: return fail(DSV_EINVAL, "unknown Pauli factor '%c'", paulis[i]);
    }
  }
  pm->h = -1;
  for (int b = 63; b >= 0; --b)
    if (pm->x >> b & 1) { pm->h = b; break; }
  return DSV_OK;
}

// (-i)^ny
void minus_i_pow(int ny, double* re, double* im) {
  static const double t[4][2] = {{1, 0}, {0, -1}, {-1, 0}, {0, 1}};
  *re = t[ny & 3][0];
  *im = t[ny & 3][1];
}

}  // namespace

extern "C" {

int dsv_config_set(const char* key, int value) {
  // the kernel-selection switches otherwise read once from the environment
  // (DSV_TC, DSV_TC8, DSV_LOW, DSV_LOWT, DSV_DBLK8, DSV_BLK8, DSV_WT)
  static const struct {
    const char* name;
    bool* flag;
  } kKeys[] = {{"tc", &g_tc_env},         {"tc8", &g_tc8_env},     {"tc8ws", &g_tc8ws_env}, {"tc8ws_all", &g_tc8ws_all}, {"tc8ws_row2", &g_tc8ws_row2},  {"tma", &g_tma_env}, {"rowvec", &g_rowvec_env}, {"tc8d", &g_tc8d_env}, {"tc8d512", &g_tc8d512}, {"tc8_pair01", &g_tc8_pair01}, {"tc8_pairswap", &g_tc8_pairswap}, {"tc4_all", &g_tc4_all},    {"low", &g_low_env}, {"lowt", &g_lowt_env},
               {"dblk8", &g_dblk8_env}, {"blk8", &g_blk8_env}, {"wt", &g_wt_env}};
  if (!key) return fail(DSV_EINVAL, "null key");
  for (const auto& k : kKeys)
    if (std::strcmp(k.name, key) == 0) {
      *k.flag = value != 0;
      return DSV_OK;
    }
  return fail(DSV_EINVAL, "unknown config key '%s'", key);
}

const char* dsv_last_error(void) { return g_err.c_str(); }
int dsv_version(void) { return 1; }

int dsv_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *out = n;
  return DSV_OK;
}

int dsv_launch_count(uint64_t* out) {
  *out = g_launches.load();
  return DSV_OK;
}

// ---- state-buffer cache ------------------------------------------------------------
// cudaMalloc / cudaFree of a 64 GiB state cost tens to hundreds of ms (measured
// 23-56 ms / 145-837 ms at n = 33), paid per circuit by every user who builds a
// fresh StateVector.  Destroyed states park their buffer here (exact size and
// device match on reuse); an allocation that fails for lack of memory first
// releases the cache.  DSV_POOL=0 disables it; dsv_pool_release() empties it.
namespace {
struct PoolEntry {
  int device;
  size_t bytes;
  void* ptr;
  // the state's private stream and scratch buffers ride along (cudaFree and
  // cudaStreamDestroy synchronise the device: ~15 ms per state otherwise)
  cudaStream_t stream;
  void* scratch;
  size_t scratch_bytes;
  void* gdata;
  size_t gdata_bytes;
};
std::mutex g_pool_mu;
std::vector<PoolEntry> g_pool;
constexpr size_t kPoolMaxEntries = 4;
const bool g_pool_env = [] {
  const char* e = std::getenv("DSV_POOL");
  return !(e && e[0] == '0');
}();

void pool_free_entry(const PoolEntry& e) {
  DeviceGuard g(e.device);
  cudaFree(e.ptr);
  if (e.scratch) cudaFree(e.scratch);
  if (e.gdata) cudaFree(e.gdata);
  if (e.stream) cudaStreamDestroy(e.stream);
}

bool pool_take(int dev, size_t bytes, PoolEntry* out) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (size_t i = 0; i < g_pool.size(); ++i)
    if (g_pool[i].device == dev && g_pool[i].bytes == bytes) {
      *out = g_pool[i];
      g_pool.erase(g_pool.begin() + long(i));
      return true;
    }
  return false;
}

void pool_put(const PoolEntry& e) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool.push_back(e);
  if (g_pool.size() > kPoolMaxEntries) {  // oldest out
    pool_free_entry(g_pool.front());
    g_pool.erase(g_pool.begin());
  }
}

void pool_release_dev(int dev) {  // dev < 0: all devices
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (size_t i = 0; i < g_pool.size();) {
    if (dev < 0 || g_pool[i].device == dev) {
      pool_free_entry(g_pool[i]);
      g_pool.erase(g_pool.begin() + long(i));
    } else {
      ++i;
    }
  }
}
}  // namespace

int dsv_pool_release(int device) {
  pool_release_dev(device);
  return DSV_OK;
}

int dsv_state_create(int device, int nbits, int dtype, dsv_state** out) {
  if (!out) return fail(DSV_EINVAL, "null out");
  *out = nullptr;
  if (nbits < 0 || nbits > DSV_MAX_BITS) return fail(DSV_EINVAL, "nbits %d outside [0, %d]", nbits, DSV_MAX_BITS);
  if (dtype != DSV_C64 && dtype != DSV_C128) return fail(DSV_EINVAL, "dtype %d not c64/c128", dtype);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(DSV_EINVAL, "device %d outside [0, %d)", device, ndev);
  DeviceGuard g(device);
  dsv_state* s = new dsv_state;
  s->device = device;
  s->nbits = nbits;
  s->dtype = dtype;
  const size_t bytes = amp_bytes(dtype) << nbits;
  cudaError_t e = cudaSuccess;
  PoolEntry pe;
  if (g_pool_env && pool_take(device, bytes, &pe)) {
    s->d = pe.ptr;
    s->stream = pe.stream;
    s->scratch = pe.scratch;
    s->scratch_bytes = pe.scratch_bytes;
    s->gdata = pe.gdata;
    s->gdata_bytes = pe.gdata_bytes;
    *out = s;
    return dsv_set_basis(s, 0);
  }
  {
    e = cudaMalloc(&s->d, bytes);
    if (e == cudaErrorMemoryAllocation) {  // cached buffers may be holding the memory
      cudaGetLastError();
      pool_release_dev(device);
      e = cudaMalloc(&s->d, bytes);
    }
  }
  if (e != cudaSuccess) {
    delete s;
    return cuda_fail(e, "cudaMalloc(state)");
  }
  e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    cudaFree(s->d);
    delete s;
    return cuda_fail(e, "cudaStreamCreate");
  }
  *out = s;
  return dsv_set_basis(s, 0);
}

int dsv_state_destroy(dsv_state* s) {
  if (!s) return DSV_OK;
  DeviceGuard g(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (auto& r : s->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : s->ev_pool) cudaEventDestroy(e);
  for (auto e : s->uev)
    if (e) cudaEventDestroy(e);
  if (s->pinned) pinned_put(s->pinned, s->pinned_n);  // reused by the next state (cudaFreeHost synchronises)
  if (s->d && s->owned && !s->ipc && !s->exported && g_pool_env) {
    pool_put({s->device, amp_bytes(s->dtype) << s->nbits, s->d, s->stream, s->scratch, s->scratch_bytes, s->gdata,
              s->gdata_bytes});
    delete s;
    return DSV_OK;
  }
  if (s->scratch) cudaFree(s->scratch);
  if (s->gdata) cudaFree(s->gdata);
  if (s->d) {
    if (s->ipc) cudaIpcCloseMemHandle(s->d);
    else if (s->owned) cudaFree(s->d);
  }
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return DSV_OK;
}

int dsv_state_info(const dsv_state* s, int* device, int* nbits, int* dtype) {
  if (int rc = check_state(s)) return rc;
  if (device) *device = s->device;
  if (nbits) *nbits = s->nbits;
  if (dtype) *dtype = s->dtype;
  return DSV_OK;
}

int dsv_state_device_ptr(const dsv_state* s, void** out) {
  if (int rc = check_state(s)) return rc;
  *out = s->d;
  return DSV_OK;
}

int dsv_sync(dsv_state* s) {
  if (int rc = no_capture(s, "dsv_sync")) return rc;
  if (int rc = check_state(s)) return rc;
  DeviceGuard g(s->device);
  CK(cudaStreamSynchronize(s->stream));
  return DSV_OK;
}

int dsv_set_zero(dsv_state* s) {
  if (int rc = check_state(s)) return rc;
  DeviceGuard g(s->device);
  CK(cudaMemsetAsync(s->d, 0, amp_bytes(s->dtype) << s->nbits, s->stream));
  return DSV_OK;
}

int dsv_set_basis(dsv_state* s, uint64_t index) {
  if (int rc = check_state(s)) return rc;
  if (index >= namps(s)) return fail(DSV_EINVAL, "basis index out of range");
  DeviceGuard g(s->device);
  CK(cudaMemsetAsync(s->d, 0, amp_bytes(s->dtype) << s->nbits, s->stream));
  if (s->dtype == DSV_C128) {
    static const double one[2] = {1.0, 0.0};
    CK(cudaMemcpyAsync(static_cast<char*>(s->d) + 16 * index, one, 16, cudaMemcpyHostToDevice, s->stream));
  } else {
    static const float one[2] = {1.0f, 0.0f};
    CK(cudaMemcpyAsync(static_cast<char*>(s->d) + 8 * index, one, 8, cudaMemcpyHostToDevice, s->stream));
  }
  return DSV_OK;
}

int dsv_upload(dsv_state* s, uint64_t begin, uint64_t count, const void* host) {
  if (int rc = no_capture(s, "dsv_upload")) return rc;
  if (int rc = check_state(s)) return rc;
  if (begin > namps(s) || count > namps(s) - begin) return fail(DSV_EINVAL, "upload range exceeds state");
  if (count == 0) return DSV_OK;
  DeviceGuard g(s->device);
  const size_t ab = amp_bytes(s->dtype);
  CK(cudaMemcpyAsync(static_cast<char*>(s->d) + ab * begin, host, ab * count, cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return DSV_OK;
}

int dsv_download(dsv_state* s, uint64_t begin, uint64_t count, void* host) {
  if (int rc = no_capture(s, "dsv_download")) return rc;
  if (int rc = check_state(s)) return rc;
  if (begin > namps(s) || count > namps(s) - begin) return fail(DSV_EINVAL, "download range exceeds state");
  if (count == 0) return DSV_OK;
  DeviceGuard g(s->device);
  const size_t ab = amp_bytes(s->dtype);
  CK(cudaMemcpyAsync(host, static_cast<const char*>(s->d) + ab * begin, ab * count, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return DSV_OK;
}

int dsv_copy(dsv_state* dst, const dsv_state* src) {
  if (int rc = no_capture(dst, "dsv_copy")) return rc;
  if (int rc = no_capture(src, "dsv_copy")) return rc;
  if (int rc = check_state(dst)) return rc;
  if (int rc = check_state(src)) return rc;
  if (dst->nbits != src->nbits || dst->dtype != src->dtype) return fail(DSV_EINVAL, "copy between states of different shape");
  DeviceGuard g(dst->device);
  if (int rc = sync_streams(dst, const_cast<dsv_state*>(src))) return rc;
  const size_t bytes = amp_bytes(dst->dtype) << dst->nbits;
  if (dst->device == src->device)
    CK(cudaMemcpyAsync(dst->d, src->d, bytes, cudaMemcpyDeviceToDevice, dst->stream));
  else
    CK(cudaMemcpyPeerAsync(dst->d, dst->device, src->d, src->device, bytes, dst->stream));
  return sync_streams(const_cast<dsv_state*>(src), dst);
}

// ---- gates -----------------------------------------------------------------------------

int dsv_apply_matrix(dsv_state* s, const void* matrix, const int32_t* targets, int k,
                     const int32_t* cb, const int32_t* cv, int nctrl) {
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (!matrix) return fail(DSV_EINVAL, "null matrix");
  GateGeom gg;
  if (int rc = validate_gate(s, targets, k, cb, cv, nctrl, &gg)) return rc;
  DeviceGuard g(s->device);
  const double bytes = 2.0 * double(amp_bytes(s->dtype)) * std::ldexp(1.0, s->nbits - nctrl);
  const uint64_t D = 1ull << k;
  // plain k = 4 stays on the CUDA cores (random unitaries at n = 33: 0.80-0.89
  // of peak, the tensor path 0.77-0.88) except on the lowest four bits (CUDA
  // cores: 2 TB/s) and with index bit 0 a target (16-byte member pairs on the
  // tensor path: (0,5,17,30) 28.0 -> 22.6 ms)
  // contiguous targets from bit 3 up: tensor path 22.7 vs 26.2 ms on a dense
  // state at n = 33 ((8,9,10,11), tools/_tc4_probe.py), 2.96-3.04 vs
  // 3.17-3.33 ms at n = 30 for (3..6), (4..7), (5..8) (tools/_lowk4.py);
  // scattered targets and contiguous ones starting at bit 1 or 2 stay on
  // the CUDA cores
  bool contig_hi = g_tc8_env && gg.tsorted[0] >= 3 && gg.nctrl == 0;
  for (int m = 1; m < k; ++m) contig_hi = contig_hi && gg.tsorted[m] == gg.tsorted[0] + m;
  const bool tc4 = k == 4 && (tc_mode(gg) == 2 || (gg.tsorted[0] == 0 && g_tc8_env) || contig_hi || g_tc4_all);
  // the digit kernels scale by the matrix's largest entry: a non-finite
  // matrix (unitary=False callers) takes the CUDA cores, which propagate
  // NaN / inf like the reference's NumPy product
  const bool finite = matrix_finite(s, matrix, k);
  if ((k == 5 || k == 6 || tc4) && finite && tc_eligible(s, gg))
    return apply_tc(s, gg, matrix, {}, PC_DENSE_TC, bytes);
  if (finite && tc8d_eligible(s, gg)) return apply_tc8d(s, gg, matrix, {}, PC_DENSE_TC, bytes);
  bool ctl_bit0 = false;
  for (int c = 0; c < nctrl; ++c) ctl_bit0 = ctl_bit0 || cb[c] == 0;
  if (g_dblk8_env && s->dtype == DSV_C64 && k >= 2 && s->nbits >= 3 && gg.holes.back() < 3 && gg.holes[0] <= 1 &&
      (nctrl == 0 || ctl_bit0)) {
    // targets and controls inside bits 0..2: the 8 x 8 block operator on one
    // 64-byte block per thread (32-byte accesses).  n = 33: (1,2) 23.0 -> 19.6 ms,
    // (0,2) 23.6 -> 19.6, (0,1,2) 21.6 -> 19.5, (1,2) controlled by bit 0 24.6 ->
    // 19.5; a control on bit 2 keeps the low kernels (they skip the unmet half: 18.5)
    std::vector<cplx<float>> m;
    canon_matrix<float>(gg, matrix, m);
    ProfTok t = prof_start(s);
    CKL(launch_dense_blk8(s->nbits, k, gg.tsorted.data(), m.data(), cb, cv, nctrl, s->d, s->stream), 1);
    prof_stop(s, t, PC_DENSE, bytes);
    return DSV_OK;
  }
  if (k >= 2 && low_eligible(s, gg)) return apply_low(s, gg, matrix, {}, PC_DENSE_LOW, bytes);
  if (g_wt_env && nctrl == 0 && k >= 1 && k <= 4 && gg.tsorted[k - 1] < 6 && s->nbits >= 10) {
    // the register path strides lanes >= 32 bytes apart here: transpose through smem
    // measured weak layouts of the register path (tools/lowsweep.py, c128_bench.py):
    // complex64 targets {1,2,3} (0.59 -> 0.95), complex128 {0,1,2} (0.60 -> 0.76),
    // complex128 k = 4 on bits 0..3
    const bool weak = (k == 3 && (s->dtype == DSV_C128 ? gg.tsorted[0] == 0 && gg.tsorted[2] == 2
                                                       : gg.tsorted[0] == 1 && gg.tsorted[2] == 3)) ||
                      (k == 4 && s->dtype == DSV_C128 && gg.tsorted[3] == 3);  // bits 0..3: 0.59 -> 0.67
    if (weak) {
      ProfTok t = prof_start(s);
      if (s->dtype == DSV_C128) {
        std::vector<cplx<double>> m;
        canon_matrix<double>(gg, matrix, m);
        CKL(launch_dense_wt(s->dtype, s->nbits, k, gg.tsorted.data(), m.data(), s->d, s->stream), 1);
      } else {
        std::vector<cplx<float>> m;
        canon_matrix<float>(gg, matrix, m);
        CKL(launch_dense_wt(s->dtype, s->nbits, k, gg.tsorted.data(), m.data(), s->d, s->stream), 1);
      }
      prof_stop(s, t, PC_DENSE_WT, bytes);
      return DSV_OK;
    }
  }
  int nlow = 0;
  for (int m = 0; m < k; ++m) nlow += gg.tsorted[m] < (s->dtype == DSV_C64 ? 4 : 3);
  if (k >= 2 && k <= 5 && nlow >= 2 && s->nbits >= 14 && !g_disable_tile) {
    // low targets: shared-memory tiles, 2^kh rows x 2^T contiguous amplitudes
    int T = 10, kh = 0;
    for (; T >= 6; --T) {
      kh = 0;
      for (int m = 0; m < k; ++m) kh += gg.tsorted[m] >= T;
      if (T + kh <= 12) break;
    }
    TileDesc d;
    std::memset(&d, 0, sizeof d);
    d.T = T;
    d.kh = kh;
    std::vector<int> holes;
    for (int b = 0; b < T; ++b) holes.push_back(b);
    std::vector<int> high;
    for (int m = 0; m < k; ++m)
      if (gg.tsorted[m] >= T) high.push_back(gg.tsorted[m]);
    uint64_t setm = 0;
    for (int c = 0; c < nctrl; ++c) {
      if (cb[c] >= T) {
        holes.push_back(cb[c]);
        if (cv[c]) setm |= 1ull << cb[c];
      } else {
        d.cmask |= 1u << cb[c];
        if (cv[c]) d.cval |= 1u << cb[c];
      }
    }
    for (int b : high) holes.push_back(b);
    std::sort(holes.begin(), holes.end());
    if (int rc = make_geom(s->nbits, holes, setm, &d.g)) return rc;
    for (int r = 0; r < (1 << kh); ++r) {
      uint64_t o = 0;
      for (int i = 0; i < kh; ++i) o |= uint64_t((r >> i) & 1) << high[i];
      d.hoff[r] = o;
    }
    int hi_i = 0;
    for (int m = 0; m < k; ++m) d.lt[m] = gg.tsorted[m] < T ? gg.tsorted[m] : T + hi_i++;
    ProfTok t = prof_start(s);
    if (s->dtype == DSV_C128) {
      std::vector<cplx<double>> m;
      canon_matrix<double>(gg, matrix, m);
      CKL(launch_dense_tile(s->dtype, k, d, m.data(), s->d, s->stream), 1);
    } else {
      std::vector<cplx<float>> m;
      canon_matrix<float>(gg, matrix, m);
      CKL(launch_dense_tile(s->dtype, k, d, m.data(), s->d, s->stream), 1);
    }
    prof_stop(s, t, PC_DENSE_TILE, bytes);
    return DSV_OK;
  }
  {
    // complex64 with index bit 0 a control: whole 16-byte units, only the
    // control's lane transformed (the scalar path uses half of every sector)
    int ctl0 = -1;
    for (int c = 0; c < nctrl; ++c)
      if (cb[c] == 0) ctl0 = cv[c];
    if (ctl0 >= 0 && s->dtype == DSV_C64 && k >= 1 && k <= 4 && s->nbits >= 2) {
      std::vector<int> h;
      for (int b : gg.holes)
        if (b != 0) h.push_back(b - 1);
      Geom geo;
      if (int rc = make_geom(s->nbits - 1, h, (gg.set_mask & ~1ull) >> 1, &geo)) return rc;
      std::vector<uint64_t> offs(D);
      for (uint64_t j = 0; j < D; ++j) {
        uint64_t o = 0;
        for (int m = 0; m < k; ++m) o |= ((j >> m) & 1ull) << (gg.tsorted[m] - 1);
        offs[j] = o;
      }
      std::vector<cplx<float>> m;
      canon_matrix<float>(gg, matrix, m);
      ProfTok t = prof_start(s);
      CKL(launch_dense_lanectl(k, geo, offs.data(), m.data(), ctl0, s->d, s->stream), 1);
      prof_stop(s, t, PC_DENSE, bytes);
      return DSV_OK;
    }
  }
  if (k <= kDenseRegMaxK) {
    UnitView uv;
    // float4 pairs only while 2^k x 2 amplitudes fit the register budget
    if (int rc = unit_view(s, gg, k <= 4, &uv)) return rc;
    ProfTok t = prof_start(s);
    if (s->dtype == DSV_C128) {
      std::vector<cplx<double>> m;
      canon_matrix<double>(gg, matrix, m);
      CKL(launch_dense_reg(s->dtype, uv.mode, k, uv.g, uv.offs.data(), m.data(), s->d, s->stream), 1);
    } else {
      std::vector<cplx<float>> m;
      canon_matrix<float>(gg, matrix, m);
      CKL(launch_dense_reg(s->dtype, uv.mode, k, uv.g, uv.offs.data(), m.data(), s->d, s->stream), 1);
    }
    prof_stop(s, t, PC_DENSE, bytes);
    return DSV_OK;
  }
  // generic path (k = 6..10): offsets + transposed matrix staged in device scratch
  UnitView uv;
  if (int rc = unit_view(s, gg, false, &uv)) return rc;
  const size_t ab = amp_bytes(s->dtype);
  const size_t off_bytes = D * sizeof(uint64_t);
  const size_t mat_bytes = D * D * ab;
  if (int rc = ensure_scratch(s, off_bytes + mat_bytes + 256)) return rc;
  std::vector<unsigned char> mt(mat_bytes);
  if (s->dtype == DSV_C128) {
    std::vector<cplx<double>> m;
    canon_matrix<double>(gg, matrix, m);
    cplx<double>* o = reinterpret_cast<cplx<double>*>(mt.data());
    for (uint64_t r = 0; r < D; ++r)
      for (uint64_t c = 0; c < D; ++c) o[c * D + r] = m[r * D + c];
  } else {
    std::vector<cplx<float>> m;
    canon_matrix<float>(gg, matrix, m);
    cplx<float>* o = reinterpret_cast<cplx<float>*>(mt.data());
    for (uint64_t r = 0; r < D; ++r)
      for (uint64_t c = 0; c < D; ++c) o[c * D + r] = m[r * D + c];
  }
  char* base = static_cast<char*>(s->scratch);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(base);
  void* d_mt = base + ((off_bytes + 255) / 256) * 256;
  CK(h2d(s, d_offs, uv.offs.data(), off_bytes));
  CK(h2d(s, d_mt, mt.data(), mat_bytes));
  ProfTok t = prof_start(s);
  CKL(launch_dense_generic(s->dtype, k, uv.g, d_offs, d_mt, s->d, s->stream), 1);
  prof_stop(s, t, PC_DENSE_GENERIC, bytes);
  // the host staging vectors die at return: make the copies complete first
  if (!s->capturing) CK(cudaStreamSynchronize(s->stream));
  return DSV_OK;
}

int dsv_apply_matrix_phased(dsv_state* s, const void* matrix, const int32_t* targets, int k,
                            const int32_t* cross_t, const int32_t* cross_b, const double* cross_theta,
                            int ncross, const int32_t* out_b, const double* out_theta, int nout) {
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (!matrix) return fail(DSV_EINVAL, "null matrix");
  if (k < 1 || k > 6) return fail(DSV_EUNSUPPORTED, "phased window arity %d outside [1, 6]", k);
  if (ncross < 0 || nout < 0) return fail(DSV_EINVAL, "negative term count");
  GateGeom gg;
  if (int rc = validate_gate(s, targets, k, nullptr, nullptr, 0, &gg)) return rc;
  uint64_t tmask = 0;
  for (int m = 0; m < k; ++m) tmask |= 1ull << targets[m];
  // sorted position of caller target index m
  std::vector<int> newpos(k);
  for (int mp = 0; mp < k; ++mp) newpos[gg.order[mp]] = mp;
  using Term = PhaseTerm;
  std::vector<Term> terms;
  for (int x = 0; x < ncross; ++x) {
    if (cross_t[x] < 0 || cross_t[x] >= k) return fail(DSV_EINVAL, "cross term target index %d out of range", cross_t[x]);
    const int b = cross_b[x];
    if (b < 0 || b >= s->nbits || (tmask >> b & 1)) return fail(DSV_EINVAL, "cross term bit %d must be an outside bit", b);
    terms.push_back({newpos[cross_t[x]], b, cross_theta[x]});
  }
  for (int y = 0; y < nout; ++y) {
    const int b = out_b[y];
    if (b < 0 || b >= s->nbits || (tmask >> b & 1)) return fail(DSV_EINVAL, "outside term bit %d must be an outside bit", b);
    terms.push_back({k, b, out_theta[y]});
  }
  DeviceGuard g(s->device);
  const bool finite = matrix_finite(s, matrix, k);
  if (finite && tc_eligible(s, gg))
    return apply_tc(s, gg, matrix, terms, PC_DENSE_TC, 2.0 * double(amp_bytes(s->dtype)) * double(namps(s)));
  if (finite && tc8d_eligible(s, gg))
    return apply_tc8d(s, gg, matrix, terms, PC_DENSE_TC, 2.0 * double(amp_bytes(s->dtype)) * double(namps(s)));
  if (k > kDenseRegMaxK)  // the host layer then applies the phases as diagonal gates
    return fail(DSV_EUNSUPPORTED, "phased 6-qubit window needs the tensor-core path (complex64, >= 7 free bits)");
  if (low_eligible(s, gg))
    return apply_low(s, gg, matrix, terms, PC_DENSE_LOW, 2.0 * double(amp_bytes(s->dtype)) * double(namps(s)));
  UnitView uv;
  if (int rc = unit_view(s, gg, k <= 4, &uv)) return rc;
  // active index bytes and the [nchunk][256][k+1] unit-factor tables
  PhasedDesc d;
  std::memset(&d, 0, sizeof d);
  d.g = uv.g;
  for (int j = 0; j < (1 << k); ++j) d.offs[j] = uv.offs[j];
  std::vector<unsigned char> raw;
  unit_factor_tables(terms, k, s->dtype == DSV_C128, &d.nchunk, d.chunk_shift, raw);
  if (d.nchunk == 0) {  // no outside terms: still valid (plain dense), keep one zero chunk
    d.nchunk = 1;
    d.chunk_shift[0] = 0;
  }
  if (int rc = ensure_gdata(s, raw.size())) return rc;
  CK(h2d(s, s->gdata, raw.data(), raw.size()));
  const double bytes = 2.0 * double(amp_bytes(s->dtype)) * double(namps(s));
  ProfTok t = prof_start(s);
  bool lowbits = k <= 4;
  for (int m2 = 0; m2 < k; ++m2) lowbits = lowbits && gg.tsorted[m2] == m2;
  if (s->dtype == DSV_C128) {
    std::vector<cplx<double>> m;
    canon_matrix<double>(gg, matrix, m);
    if (g_lowt_env && lowbits && s->nbits >= 12)  // warp-transposed runs: coalesced 16-byte units
      CKL(launch_dense_lowt128(k, !terms.empty(), d, namps(s), m.data(), s->gdata, s->d, s->stream), 1);
    else
      CKL(launch_dense_phased(s->dtype, uv.mode, k, d, m.data(), s->gdata, s->d, s->stream), 1);
  } else {
    std::vector<cplx<float>> m;
    canon_matrix<float>(gg, matrix, m);
    CKL(launch_dense_phased(s->dtype, uv.mode, k, d, m.data(), s->gdata, s->d, s->stream), 1);
  }
  prof_stop(s, t, PC_DENSE_PHASED, bytes);
  return DSV_OK;
}

int dsv_apply_genperm(dsv_state* s, const int64_t* perm, const void* diag, const int32_t* targets,
                      int k, const int32_t* cb, const int32_t* cv, int nctrl) {
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (!perm || !diag) return fail(DSV_EINVAL, "null permutation/diagonal");
  GateGeom gg;
  if (int rc = validate_gate(s, targets, k, cb, cv, nctrl, &gg)) return rc;
  const uint64_t D = 1ull << k;
  {
    std::vector<char> hit(D, 0);
    for (uint64_t j = 0; j < D; ++j) {
      if (perm[j] < 0 || uint64_t(perm[j]) >= D || hit[perm[j]])
        return fail(DSV_EINVAL, "permutation table is not a bijection");
      hit[perm[j]] = 1;
    }
  }
  DeviceGuard g(s->device);
  // canonical tables: perm'[j'] = new(perm[old(j')]), diag'[j'] = diag[old(j')]
  std::vector<uint64_t> pn(D);
  std::vector<unsigned char> dn(D * amp_bytes(s->dtype));
  uint64_t nactive = 0;
  std::vector<char> act(D, 0);
  for (uint64_t jn = 0; jn < D; ++jn) {
    const uint64_t j = old_index(gg, jn);
    pn[jn] = new_index(gg, uint64_t(perm[j]));
    bool unit;
    if (s->dtype == DSV_C128) {
      const cplx<double> v = static_cast<const cplx<double>*>(diag)[j];
      reinterpret_cast<cplx<double>*>(dn.data())[jn] = v;
      unit = v.x == 1.0 && v.y == 0.0;
    } else {
      const cplx<float> v = static_cast<const cplx<float>*>(diag)[j];
      reinterpret_cast<cplx<float>*>(dn.data())[jn] = v;
      unit = v.x == 1.0f && v.y == 0.0f;
    }
    act[jn] = !(pn[jn] == jn && unit);
    nactive += act[jn];
  }
  if (nactive == 0) return DSV_OK;  // identity table: nothing moves (bit-exact no-op)
  const double bytes = 2.0 * double(amp_bytes(s->dtype)) * std::ldexp(1.0, s->nbits - nctrl) *
                       double(nactive) / double(D);
  bool is_diag = true;
  for (uint64_t j = 0; j < D; ++j) is_diag = is_diag && pn[j] == j;
  const int kk = k + nctrl;
  if (g_blk8_env && s->dtype == DSV_C64 && s->nbits >= 3 && k >= 1 && gg.holes.back() < 3 && gg.holes[0] <= 1 &&
      (nctrl == 0 || is_diag || gg.holes[0] == 0)) {
    // targets and controls inside bits 0..2, touching bit 0 or 1 (CP(0, 1),
    // SWAP(0, 1), 2-3 qubit permutations on the lowest bits ...): every group
    // inside one 64-byte block, one full pass with full-sector 32-byte accesses
    // (n = 33: 22-25 -> 19.7 ms).  Kept on the other kernels: holes = {2} alone
    // and permutations controlled above bit 0 (CX(2, 1): 16.1 ms there), whose
    // 32-byte runs let the untouched half skip its writes.
    uint64_t active = 0;
    for (uint64_t j = 0; j < D; ++j)
      if (act[j]) active |= 1ull << j;
    ProfTok t = prof_start(s);
    CKL(launch_perm_blk8(s->nbits, k, gg.tsorted.data(), pn.data(), dn.data(), active, cb, cv, nctrl, s->d,
                         s->stream), 1);
    prof_stop(s, t, PC_PERM, bytes);
    return DSV_OK;
  }
  if (is_diag && nactive == 1 && s->dtype == DSV_C64 && s->nbits >= 2 && !gg.holes.empty() && gg.holes[0] == 0 &&
      (gg.holes.size() < 2 || gg.holes[1] >= 2)) {  // (bit 1 fixed too: units 32 B apart, the stream kernel wins)
    // the same with index bit 0 fixed (target or control): 16-byte units over
    // the other bits, only the lane with bit 0's value is scaled
    uint64_t ja = 0;
    for (uint64_t j = 0; j < D; ++j)
      if (act[j]) ja = j;
    uint64_t forced = gg.set_mask;
    for (int m = 0; m < k; ++m)
      if ((ja >> m) & 1) forced |= 1ull << gg.tsorted[m];
    const int lane = int(forced & 1ull);
    std::vector<int> h;
    for (int b : gg.holes)
      if (b != 0) h.push_back(b - 1);
    Geom geo;
    if (int rc = make_geom(s->nbits - 1, h, (forced & ~1ull) >> 1, &geo)) return rc;
    const size_t es = amp_bytes(s->dtype);
    std::vector<unsigned char> d1(es);
    std::memcpy(d1.data(), dn.data() + ja * es, es);
    ProfTok t = prof_start(s);
    CKL(launch_diag_lane(geo, d1.data(), lane, s->d, s->stream), 1);
    prof_stop(s, t, PC_DIAG, bytes);
    return DSV_OK;
  }
  if (is_diag && nactive == 1 && s->dtype == DSV_C64 && !(!gg.holes.empty() && gg.holes[0] == 0) &&
      s->nbits >= 1) {
    // one non-unit entry (controlled phase, CZ, T on a control subcube ...):
    // every target and control bit is fixed, so enumerate exactly the
    // amplitudes it scales (holes = targets + controls, forced to the entry's
    // bits) and multiply in contiguous 16-byte runs; no table, no skipped work
    uint64_t ja = 0;
    for (uint64_t j = 0; j < D; ++j)
      if (act[j]) ja = j;
    uint64_t forced = gg.set_mask;  // control values (amp space)
    for (int m = 0; m < k; ++m)
      if ((ja >> m) & 1) forced |= 1ull << gg.tsorted[m];
    // (complex64 with bit 0 free only: 16-byte units; with bit 0 fixed the
    // affected amplitudes sit 16 bytes apart and the sector-skipping stream
    // kernel below is faster)
    const bool vec2 = true;
    const int sh = 1;
    std::vector<int> h(gg.holes);
    for (int& x : h) x -= sh;
    Geom geo;
    if (int rc = make_geom(s->nbits - sh, h, forced >> sh, &geo)) return rc;
    const size_t es = amp_bytes(s->dtype);
    std::vector<unsigned char> d1(es);
    std::memcpy(d1.data(), dn.data() + ja * es, es);
    const unsigned char one = 1;
    ProfTok t = prof_start(s);
    CKL(launch_diag(s->dtype, vec2 ? MODE_VEC2 : MODE_SCALAR, 0, geo, nullptr, d1.data(), &one, s->d, s->stream), 1);
    prof_stop(s, t, PC_DIAG, bytes);
    return DSV_OK;
  }
  if (is_diag && kk <= (s->dtype == DSV_C64 ? kDiagStreamMaxBits : kDiagStreamMaxBits - 1)) {
    // streaming path: one table over targets + controls, contiguous 16-B units
    std::vector<int> B(gg.holes);  // sorted targets + controls (amp bits)
    const uint64_t T = 1ull << kk;
    const size_t es = amp_bytes(s->dtype);
    std::vector<unsigned char> tab((es + 1) * T);
    unsigned char* fl = tab.data() + es * T;
    std::vector<int> pos_t(k), pos_c(nctrl);
    for (int m = 0; m < k; ++m) pos_t[m] = int(std::find(B.begin(), B.end(), gg.tsorted[m]) - B.begin());
    for (int c = 0; c < nctrl; ++c) pos_c[c] = int(std::find(B.begin(), B.end(), cb[c]) - B.begin());
    for (uint64_t x = 0; x < T; ++x) {
      bool ok = true;
      for (int c = 0; c < nctrl; ++c) ok = ok && int((x >> pos_c[c]) & 1ull) == cv[c];
      uint64_t j = 0;
      for (int m = 0; m < k; ++m) j |= ((x >> pos_t[m]) & 1ull) << m;
      if (s->dtype == DSV_C128) {
        reinterpret_cast<cplx<double>*>(tab.data())[x] =
            ok ? reinterpret_cast<const cplx<double>*>(dn.data())[j] : cplx<double>{1.0, 0.0};
      } else {
        reinterpret_cast<cplx<float>*>(tab.data())[x] =
            ok ? reinterpret_cast<const cplx<float>*>(dn.data())[j] : cplx<float>{1.0f, 0.0f};
      }
      fl[x] = (ok && act[j]) ? 1 : 0;
    }
    // a 32-byte sector spans amp bits {0,1} (complex64) or {0} (complex128)
    uint64_t smask = 0;
    for (int m = 0; m < kk; ++m)
      if (B[m] < (s->dtype == DSV_C64 ? 2 : 1)) smask |= 1ull << m;
    for (uint64_t x = 0; x < T; ++x) {
      bool touched = false;
      for (uint64_t sub = smask;; sub = (sub - 1) & smask) {
        touched = touched || (fl[x ^ sub] & 1);
        if (!sub) break;
      }
      if (touched) fl[x] |= 2;
    }
    if (int rc = ensure_gdata(s, tab.size())) return rc;
    CK(h2d(s, s->gdata, tab.data(), tab.size()));
    ProfTok t = prof_start(s);
    CKL(launch_diag_stream(s->dtype, s->nbits, kk, B.data(), s->gdata, s->d, s->stream), 1);
    prof_stop(s, t, PC_DIAG, bytes);
    return DSV_OK;
  }
  if (is_diag) {
    // elementwise path: holes = control bits only, targets stay in the stream
    GateGeom cg = gg;
    cg.holes.clear();
    for (int c = 0; c < nctrl; ++c) cg.holes.push_back(cb[c]);
    std::sort(cg.holes.begin(), cg.holes.end());
    const bool bit0_used = (!gg.tsorted.empty() && gg.tsorted[0] == 0) || (!cg.holes.empty() && cg.holes[0] == 0);
    const bool vec2 = s->dtype == DSV_C64 && !bit0_used && s->nbits >= 1;
    const int sh = vec2 ? 1 : 0;
    std::vector<int> h(cg.holes);
    for (int& x : h) x -= sh;
    Geom geo;
    if (int rc = make_geom(s->nbits - sh, h, gg.set_mask >> sh, &geo)) return rc;
    int tb[DSV_MAX_TARGETS];
    for (int m = 0; m < k; ++m) tb[m] = gg.tsorted[m] - sh;
    std::vector<unsigned char> av(D);
    for (uint64_t j = 0; j < D; ++j) av[j] = act[j];
    ProfTok t = prof_start(s);
    CKL(launch_diag(s->dtype, vec2 ? MODE_VEC2 : MODE_SCALAR, k, geo, tb, dn.data(), av.data(), s->d, s->stream), 1);
    prof_stop(s, t, PC_PERM, bytes);
    return DSV_OK;
  }
  if (g_wt_env && nctrl == 0 && k >= 1 && k <= (s->dtype == DSV_C128 ? 3 : 4) && gg.tsorted[k - 1] < 6 &&
      gg.tsorted[0] <= 1 && s->nbits >= 10) {
    // targets on index bits 0/1 and all below 6: the register path's lanes sit
    // >= 32 bytes apart (perm2 on (0,1) measured 0.59): warp-transposed runs
    uint64_t active = 0;
    for (uint64_t j = 0; j < D; ++j)
      if (act[j]) active |= 1ull << j;
    ProfTok t = prof_start(s);
    CKL(launch_perm_wt(s->dtype, s->nbits, k, gg.tsorted.data(), pn.data(), dn.data(), active, s->d, s->stream), 1);
    prof_stop(s, t, PC_PERM, bytes);
    return DSV_OK;
  }
  // complex64, index bit 0 a control (e.g. CNOT controlled by qubit 0): the
  // affected amplitudes sit 16 bytes apart; move whole 16-byte units over the
  // other bits and let only the control's lane change (full sectors instead of
  // half-used ones)
  int ctl0 = -1;
  for (int c = 0; c < nctrl; ++c)
    if (cb[c] == 0) ctl0 = cv[c];
  if (ctl0 >= 0 && s->dtype == DSV_C64 && k >= 1 && k <= 4 && s->nbits >= 2) {
    std::vector<int> h;
    for (int b : gg.holes)
      if (b != 0) h.push_back(b - 1);
    Geom geo;
    if (int rc = make_geom(s->nbits - 1, h, (gg.set_mask & ~1ull) >> 1, &geo)) return rc;
    std::vector<uint64_t> oi(D), oo(D);
    std::vector<uint8_t> pd(D);
    for (uint64_t j = 0; j < D; ++j) {
      uint64_t o = 0;
      for (int m = 0; m < k; ++m) o |= ((j >> m) & 1ull) << (gg.tsorted[m] - 1);
      oi[j] = o;
    }
    uint64_t active = 0;
    for (uint64_t j = 0; j < D; ++j) {
      oo[j] = oi[pn[j]];
      pd[j] = uint8_t(pn[j]);
      if (act[j]) active |= 1ull << j;
    }
    ProfTok t = prof_start(s);
    CKL(launch_perm_lanectl(k, geo, oi.data(), oo.data(), dn.data(), active, ctl0, pd.data(), s->d, s->stream), 1);
    prof_stop(s, t, PC_PERM, bytes);
    return DSV_OK;
  }
  if (k <= kPermRegMaxK) {
    UnitView uv;
    if (int rc = unit_view(s, gg, k <= 4, &uv)) return rc;
    std::vector<uint64_t> oo(D);
    uint64_t active = 0;
    for (uint64_t j = 0; j < D; ++j) {
      oo[j] = uv.offs[pn[j]];
      if (act[j]) active |= 1ull << j;
    }
    ProfTok t = prof_start(s);
    CKL(launch_perm_reg(s->dtype, uv.mode, k, uv.g, uv.offs.data(), oo.data(), dn.data(), active, s->d, s->stream), 1);
    prof_stop(s, t, PC_PERM, bytes);
    return DSV_OK;
  }
  UnitView uv;
  if (int rc = unit_view(s, gg, false, &uv)) return rc;
  std::vector<uint64_t> oo(D);
  for (uint64_t j = 0; j < D; ++j) oo[j] = uv.offs[pn[j]];
  const size_t ob = D * sizeof(uint64_t);
  const size_t obr = ((ob + 255) / 256) * 256;
  if (int rc = ensure_scratch(s, 2 * obr + dn.size() + 256)) return rc;
  char* base = static_cast<char*>(s->scratch);
  CK(h2d(s, base, uv.offs.data(), ob));
  CK(h2d(s, base + obr, oo.data(), ob));
  CK(h2d(s, base + 2 * obr, dn.data(), dn.size()));
  ProfTok t = prof_start(s);
  CKL(launch_perm_generic(s->dtype, k, uv.g, reinterpret_cast<uint64_t*>(base),
                          reinterpret_cast<uint64_t*>(base + obr), base + 2 * obr, s->d, s->stream), 1);
  prof_stop(s, t, PC_PERM_GENERIC, bytes);
  if (!s->capturing) CK(cudaStreamSynchronize(s->stream));
  return DSV_OK;
}

int dsv_apply_pauli_rotation(dsv_state* s, double theta, double coef_re, double coef_im,
                             const int32_t* bits, const char* paulis, int m) {
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  PauliMasks pm;
  if (int rc = parse_pauli(s, bits, paulis, m, &pm)) return rc;
  DeviceGuard g(s->device);
  double pr, pi;
  minus_i_pow(pm.ny, &pr, &pi);
  const double sn = std::sin(theta / 2), cs = std::cos(theta / 2);
  // B = -i * sin * coef * (-i)^ny
  const double cr = coef_re * pr - coef_im * pi, ci = coef_re * pi + coef_im * pr;
  PauliOp op;
  op.xmask = pm.x;
  op.yzmask = pm.yz;
  op.hbit = pm.h;
  op.c = cs;
  op.br = sn * ci;
  op.bi = -sn * cr;
  ProfTok t = prof_start(s);
  CKL(launch_pauli(s->dtype, s->nbits, op, s->d, s->stream), 1);
  prof_stop(s, t, PC_PAULI, 2.0 * double(amp_bytes(s->dtype)) * double(namps(s)));
  return DSV_OK;
}

int dsv_apply_pauli_product(dsv_state* s, const int32_t* bits, const char* paulis, int m) {
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  PauliMasks pm;
  if (int rc = parse_pauli(s, bits, paulis, m, &pm)) return rc;
  if (pm.x == 0 && pm.yz == 0) return DSV_OK;
  DeviceGuard g(s->device);
  PauliOp op;
  op.xmask = pm.x;
  op.yzmask = pm.yz;
  op.hbit = pm.h;
  op.c = 0.0;
  minus_i_pow(pm.ny, &op.br, &op.bi);
  ProfTok t = prof_start(s);
  CKL(launch_pauli(s->dtype, s->nbits, op, s->d, s->stream), 1);
  prof_stop(s, t, PC_PAULI, 2.0 * double(amp_bytes(s->dtype)) * double(namps(s)));
  return DSV_OK;
}

// ---- layout -----------------------------------------------------------------------------

int dsv_swap_index_bits(dsv_state* s, const int32_t* pairs, int npairs) {
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (npairs < 0) return fail(DSV_EINVAL, "negative pair count");
  uint64_t seen = 0;
  SwapPairs sp;
  sp.np = 0;
  bool bit0 = false;
  for (int q = 0; q < npairs; ++q) {
    const int a = pairs[2 * q], b = pairs[2 * q + 1];
    if (a < 0 || a >= s->nbits || b < 0 || b >= s->nbits)
      return fail(DSV_EINVAL, "bit pair (%d, %d) exceeds %d qubits", a, b, s->nbits);
    if ((seen >> a & 1) || (seen >> b & 1) || (a == b && false))
      return fail(DSV_EINVAL, "bit appears in more than one pair");
    seen |= 1ull << a;
    seen |= 1ull << b;
    if (a == b) continue;
    if (sp.np >= 20) return fail(DSV_EUNSUPPORTED, "more than 20 swap pairs");
    sp.a[sp.np] = a;
    sp.b[sp.np] = b;
    sp.np++;
    if (a == 0 || b == 0) bit0 = true;
  }
  if (sp.np == 0) return DSV_OK;
  DeviceGuard g(s->device);
  if (sp.np == 1 && bit0 && s->dtype == DSV_C64 && s->nbits >= 2) {
    const int b = sp.a[0] == 0 ? sp.b[0] : sp.a[0];
    ProfTok t = prof_start(s);
    CKL(launch_swap_bit0(s->nbits, b, s->d, s->stream), 1);
    prof_stop(s, t, PC_SWAP, double(amp_bytes(s->dtype)) * double(namps(s)));
    return DSV_OK;
  }
  int mode = MODE_SCALAR;
  uint64_t nunits = namps(s);
  if (s->dtype == DSV_C64 && !bit0) {
    mode = MODE_VEC2;
    nunits >>= 1;
    for (int q = 0; q < sp.np; ++q) { sp.a[q] -= 1; sp.b[q] -= 1; }
  }
  const double bytes = 2.0 * double(amp_bytes(s->dtype)) * double(namps(s)) * (1.0 - std::ldexp(1.0, -sp.np));
  const int ubits = s->nbits - (mode == MODE_VEC2 ? 1 : 0);
  if (sp.np <= 3 && ubits - 2 * sp.np >= 0) {
    SwapGeomP gp;
    std::memset(&gp, 0, sizeof gp);
    std::vector<int> holes;
    for (int q = 0; q < sp.np; ++q) {
      holes.push_back(sp.a[q]);
      holes.push_back(sp.b[q]);
    }
    std::sort(holes.begin(), holes.end());
    if (int rc = make_geom(ubits, holes, 0, &gp.g)) return rc;
    for (uint32_t pat = 0; pat < (1u << (2 * sp.np)); ++pat) {
      uint64_t i = 0, j = 0;
      for (int q = 0; q < sp.np; ++q) {
        const uint64_t xa = pat >> (2 * q) & 1, xb = pat >> (2 * q + 1) & 1;
        i |= xa << sp.a[q] | xb << sp.b[q];
        j |= xb << sp.a[q] | xa << sp.b[q];  // the pair's two bits exchanged
      }
      if (j > i) {
        gp.oi[gp.nsw] = i;
        gp.oj[gp.nsw] = j;
        ++gp.nsw;
      }
    }
    ProfTok t = prof_start(s);
    CKL(launch_swap_geom(s->dtype, mode, gp, s->d, s->stream), 1);
    prof_stop(s, t, PC_SWAP, bytes);
    return DSV_OK;
  }
  ProfTok t = prof_start(s);
  CKL(launch_swap_bits(s->dtype, mode, nunits, sp, s->d, s->stream), 1);
  prof_stop(s, t, PC_SWAP, bytes);
  return DSV_OK;
}

static int check_ordering(const dsv_state* s, const int32_t* ordering) {
  uint64_t seen = 0;
  for (int b = 0; b < s->nbits; ++b) {
    const int o = ordering[b];
    if (o < 0 || o >= s->nbits || (seen >> o & 1))
      return fail(DSV_EINVAL, "bit_ordering must be a permutation of all index bits");
    seen |= 1ull << o;
  }
  return DSV_OK;
}

static const uint64_t kAccessChunk = 1ull << 25;

int dsv_access_get(dsv_state* s, const int32_t* ordering, uint64_t begin, uint64_t end, void* host_out) {
  if (int rc = no_capture(s, "dsv_access_get")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (int rc = check_ordering(s, ordering)) return rc;
  if (!(begin < end && end <= namps(s))) return fail(DSV_EINVAL, "bad range [%llu, %llu)",
                                                     (unsigned long long)begin, (unsigned long long)end);
  DeviceGuard g(s->device);
  const size_t ab = amp_bytes(s->dtype);
  const uint64_t chunk = std::min<uint64_t>(end - begin, kAccessChunk);
  if (int rc = ensure_scratch(s, chunk * ab)) return rc;
  for (uint64_t b0 = begin; b0 < end; b0 += chunk) {
    const uint64_t cnt = std::min<uint64_t>(chunk, end - b0);
    ProfTok t = prof_start(s);
    CKL(launch_gather(s->dtype, s->nbits, ordering, b0, cnt, s->d, s->scratch, s->stream), 1);
    prof_stop(s, t, PC_ACCESS, 2.0 * ab * cnt);
    CK(cudaMemcpyAsync(static_cast<char*>(host_out) + (b0 - begin) * ab, s->scratch, cnt * ab,
                       cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  }
  return DSV_OK;
}

int dsv_access_set(dsv_state* s, const int32_t* ordering, uint64_t begin, uint64_t count, const void* host_in) {
  if (int rc = no_capture(s, "dsv_access_set")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (int rc = check_ordering(s, ordering)) return rc;
  if (count == 0 || begin >= namps(s) || count > namps(s) - begin) return fail(DSV_EINVAL, "range exceeds state size");
  DeviceGuard g(s->device);
  const size_t ab = amp_bytes(s->dtype);
  const uint64_t chunk = std::min<uint64_t>(count, kAccessChunk);
  if (int rc = ensure_scratch(s, chunk * ab)) return rc;
  for (uint64_t o = 0; o < count; o += chunk) {
    const uint64_t cnt = std::min<uint64_t>(chunk, count - o);
    CK(cudaMemcpyAsync(s->scratch, static_cast<const char*>(host_in) + o * ab, cnt * ab,
                       cudaMemcpyHostToDevice, s->stream));
    ProfTok t = prof_start(s);
    CKL(launch_scatter(s->dtype, s->nbits, ordering, begin + o, cnt, s->d, s->scratch, s->stream), 1);
    prof_stop(s, t, PC_ACCESS, 2.0 * ab * cnt);
    CK(cudaStreamSynchronize(s->stream));
  }
  return DSV_OK;
}

// ---- reductions -----------------------------------------------------------------------------

static int probs_impl(dsv_state* s, const int32_t* bits, int k, bool allow_vec2, double* host_out,
                      double** d_partial_out, uint64_t* nchunks_out, uint64_t* chunk_amps_out = nullptr) {
  if (k < 0 || k > 26) return fail(DSV_EUNSUPPORTED, "marginal over %d bits not supported (max 26)", k);
  uint64_t seen = 0;
  for (int j = 0; j < k; ++j) {
    const int b = bits[j];
    if (b < 0 || b >= s->nbits) return fail(DSV_EINVAL, "qubit bit %d out of range", b);
    if (seen >> b & 1) return fail(DSV_EINVAL, "qubits must be distinct");
    seen |= 1ull << b;
  }
  {  // inner (per-thread) / outer (block-grid) split of the binned bits
    const int ib_bits = s->dtype == DSV_C64 ? 9 : 8;  // amp bits held by (unit lane, thread index)
    const int shift1 = s->dtype == DSV_C64 ? 1 : 0;
    InnerBins ib;
    std::memset(&ib, 0, sizeof ib);
    BinGeom bg1;
    std::memset(&bg1, 0, sizeof bg1);
    bg1.reg_j = -1;
    std::vector<int> oholes;
    // (chunk partials for sampling: only without binning, where chunk c is
    // the amplitude-contiguous run of kReduceThreads * kReduceUnitsPerThread units)
    bool ok = s->nbits >= ib_bits && (d_partial_out == nullptr || (k == 0 && chunk_amps_out));
    for (int j = 0; j < k && ok; ++j) {
      const int b = bits[j];
      if (b < ib_bits) {
        if (ib.n >= 8) {
          ok = false;
          break;
        }
        ib.pos[ib.n] = b;
        ib.fin[ib.n++] = j;
        if (s->dtype == DSV_C64) {
          if (b == 0) ib.h_binned = 1;
          else if (b <= 5) ib.lane_mask |= 1u << (b - 1);
          else ib.warp_mask |= 1u << (b - 6);
        } else {
          if (b <= 4) ib.lane_mask |= 1u << b;
          else ib.warp_mask |= 1u << (b - 5);
        }
      } else {
        ib.ofin[bg1.nb] = j;
        bg1.bits[bg1.nb++] = b - shift1;
        oholes.push_back(b - shift1);
      }
    }
    if (ok) {
      std::sort(oholes.begin(), oholes.end());
      if (int rc = make_geom(s->nbits - shift1, oholes, 0, &bg1.g)) return rc;
      bg1.nchunks = chunks_for(bg1.g.nwork);
      const uint64_t nbins = 1ull << k;
      const size_t part_bytes = sizeof(double) * nbins * bg1.nchunks;
      const size_t part_round = ((part_bytes + 255) / 256) * 256;
      if (int rc = ensure_scratch(s, part_round + sizeof(double) * nbins)) return rc;
      double* d_partial = static_cast<double*>(s->scratch);
      double* d_out = reinterpret_cast<double*>(static_cast<char*>(s->scratch) + part_round);
      ProfTok t = prof_start(s);
      CKL(launch_probs_in(s->dtype, bg1, ib, s->d, d_partial, s->stream), 1);
      prof_stop(s, t, PC_REDUCE, double(amp_bytes(s->dtype)) * double(namps(s)));
      if (d_partial_out) {
        *d_partial_out = d_partial;
        *nchunks_out = bg1.nchunks;
        *chunk_amps_out = uint64_t(kReduceThreads) * kReduceUnitsPerThread * (s->dtype == DSV_C64 ? 2 : 1);
        return DSV_OK;
      }
      return finish_reduce(s, nbins, bg1.nchunks, 1, d_partial, d_out, host_out);
    }
  }
  // complex64 with bit 0 binned: float4 units, bit 0 resolved in registers
  const bool reg0 = s->dtype == DSV_C64 && (seen & 1ull) && s->nbits >= 1;
  const bool vec2 = (allow_vec2 && s->dtype == DSV_C64 && !(seen & 1ull) && s->nbits >= 1) || reg0;
  const int shift = vec2 ? 1 : 0;
  BinGeom bg;
  std::memset(&bg, 0, sizeof bg);
  bg.reg_j = -1;
  std::vector<int> holes;
  for (int b = reg0 ? 1 : 0; b < 64; ++b)
    if (seen >> b & 1) holes.push_back(b - shift);
  if (int rc = make_geom(s->nbits - shift, holes, 0, &bg.g)) return rc;
  bg.nb = 0;
  for (int j = 0; j < k; ++j) {
    if (reg0 && bits[j] == 0) {
      bg.reg_j = j;
      continue;
    }
    bg.bits[bg.nb++] = bits[j] - shift;
  }
  bg.nchunks = chunks_for(bg.g.nwork);
  const uint64_t nbins = 1ull << k;
  const size_t part_bytes = sizeof(double) * nbins * bg.nchunks;
  const size_t part_round = ((part_bytes + 255) / 256) * 256;
  if (int rc = ensure_scratch(s, part_round + sizeof(double) * nbins)) return rc;
  double* d_partial = static_cast<double*>(s->scratch);
  double* d_out = reinterpret_cast<double*>(static_cast<char*>(s->scratch) + part_round);
  ProfTok t = prof_start(s);
  CKL(launch_probs(s->dtype, vec2 ? MODE_VEC2 : MODE_SCALAR, bg, s->d, d_partial, s->stream), 1);
  prof_stop(s, t, PC_REDUCE, double(amp_bytes(s->dtype)) * double(namps(s)));
  if (d_partial_out) {
    *d_partial_out = d_partial;
    *nchunks_out = bg.nchunks;
    return DSV_OK;
  }
  return finish_reduce(s, nbins, bg.nchunks, 1, d_partial, d_out, host_out);
}

int dsv_norm2(dsv_state* s, double* out) {
  if (int rc = no_capture(s, "dsv_norm2")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  DeviceGuard g(s->device);
  return probs_impl(s, nullptr, 0, true, out, nullptr, nullptr);
}

int dsv_marginal_probs(dsv_state* s, const int32_t* bits, int k, double* out) {
  if (int rc = no_capture(s, "dsv_marginal_probs")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  DeviceGuard g(s->device);
  return probs_impl(s, bits, k, true, out, nullptr, nullptr);
}

int dsv_expect_pauli(dsv_state* s, const int32_t* bits, const char* paulis, int m, double* out) {
  if (int rc = no_capture(s, "dsv_expect_pauli")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  PauliMasks pm;
  if (int rc = parse_pauli(s, bits, paulis, m, &pm)) return rc;
  DeviceGuard g(s->device);
  PauliOp op;
  op.xmask = pm.x;
  op.yzmask = pm.yz;
  op.hbit = pm.h;
  op.c = 0.0;
  minus_i_pow(pm.ny, &op.br, &op.bi);
  const uint64_t npairs = pm.h >= 0 ? namps(s) / 2 : namps(s);
  const uint64_t nch = chunks_for(npairs);
  const size_t pr = ((sizeof(double) * 2 * nch + 255) / 256) * 256;
  if (int rc = ensure_scratch(s, pr + 16)) return rc;
  double* d_partial = static_cast<double*>(s->scratch);
  double* d_out = reinterpret_cast<double*>(static_cast<char*>(s->scratch) + pr);
  uint64_t nchunks = 0;
  ProfTok t = prof_start(s);
  CKL(launch_expect_pauli(s->dtype, s->nbits, op, s->d, d_partial, &nchunks, s->stream), 1);
  prof_stop(s, t, PC_EXPECT, double(amp_bytes(s->dtype)) * double(namps(s)));
  return finish_reduce(s, 1, nchunks, 2, d_partial, d_out, out);
}

int dsv_inner(dsv_state* a, const dsv_state* b, double* out) {
  if (int rc = no_capture(a, "dsv_inner")) return rc;
  if (int rc = no_capture(b, "dsv_inner")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(a)) return rc;
  if (int rc = check_state(b)) return rc;
  if (a->nbits != b->nbits || a->dtype != b->dtype) return fail(DSV_EINVAL, "inner product of states with different shape");
  DeviceGuard g(a->device);
  if (a->device != b->device)
    if (int rc = enable_peer(a->device, b->device)) return rc;
  if (int rc = sync_streams(a, const_cast<dsv_state*>(b))) return rc;
  const uint64_t nch = chunks_for(namps(a));
  const size_t pr = ((sizeof(double) * 2 * nch + 255) / 256) * 256;
  if (int rc = ensure_scratch(a, pr + 16)) return rc;
  double* d_partial = static_cast<double*>(a->scratch);
  double* d_out = reinterpret_cast<double*>(static_cast<char*>(a->scratch) + pr);
  uint64_t nchunks = 0;
  ProfTok t = prof_start(a);
  CKL(launch_inner(a->dtype, namps(a), a->d, b->d, d_partial, &nchunks, a->stream), 1);
  prof_stop(a, t, PC_EXPECT, 2.0 * double(amp_bytes(a->dtype)) * double(namps(a)));
  return finish_reduce(a, 1, nchunks, 2, d_partial, d_out, out);
}

int dsv_expect_matrix(dsv_state* s, const void* matrix, const int32_t* targets, int k, double* out) {
  if (int rc = no_capture(s, "dsv_expect_matrix")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (!matrix) return fail(DSV_EINVAL, "null matrix");
  GateGeom gg;
  if (int rc = validate_gate(s, targets, k, nullptr, nullptr, 0, &gg)) return rc;
  DeviceGuard g(s->device);
  if (k <= 4) {
    UnitView uv;
    // 16-byte units (two groups per thread) when bit 0 is free, up to k = 3
    // (k = 4 with two groups per thread exceeds the register file)
    if (int rc = unit_view(s, gg, k <= 3, &uv)) return rc;
    const uint64_t maxch = 148ull * 8;
    const size_t pr = ((sizeof(double) * 2 * maxch + 255) / 256) * 256;
    if (int rc = ensure_scratch(s, pr + 16)) return rc;
    double* d_partial = static_cast<double*>(s->scratch);
    double* d_out = reinterpret_cast<double*>(static_cast<char*>(s->scratch) + pr);
    uint64_t nchunks = 0;
    ProfTok t = prof_start(s);
    if (s->dtype == DSV_C128) {
      std::vector<cplx<double>> m;
      canon_matrix<double>(gg, matrix, m);
      CKL(launch_expect_dense(s->dtype, uv.mode, k, uv.g, uv.offs.data(), m.data(), s->d, d_partial, &nchunks, s->stream), 1);
    } else {
      std::vector<cplx<float>> m;
      canon_matrix<float>(gg, matrix, m);
      CKL(launch_expect_dense(s->dtype, uv.mode, k, uv.g, uv.offs.data(), m.data(), s->d, d_partial, &nchunks, s->stream), 1);
    }
    prof_stop(s, t, PC_EXPECT, double(amp_bytes(s->dtype)) * double(namps(s)));
    return finish_reduce(s, 1, nchunks, 2, d_partial, d_out, out);
  }
  // larger observables: copy, apply, <psi|work> (the reference's own algorithm)
  dsv_state* work = nullptr;
  if (int rc = dsv_state_create(s->device, s->nbits, s->dtype, &work)) return rc;
  int rc = dsv_copy(work, s);
  if (!rc) rc = dsv_apply_matrix(work, matrix, targets, k, nullptr, nullptr, 0);
  if (!rc) rc = sync_streams(s, work);
  if (!rc) rc = dsv_inner(s, work, out);
  dsv_state_destroy(work);
  return rc;
}

int dsv_collapse(dsv_state* s, const int32_t* bits, int k, uint64_t outcome, double norm2_kept) {
  if (int rc = no_capture(s, "dsv_collapse")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (!(norm2_kept > 0.0)) return fail(DSV_EINVAL, "collapse onto a zero-probability outcome");
  uint64_t mask = 0, val = 0;
  for (int j = 0; j < k; ++j) {
    const int b = bits[j];
    if (b < 0 || b >= s->nbits) return fail(DSV_EINVAL, "qubit bit %d out of range", b);
    if (mask >> b & 1) return fail(DSV_EINVAL, "qubits must be distinct");
    mask |= 1ull << b;
    val |= ((outcome >> j) & 1ull) << b;
  }
  DeviceGuard g(s->device);
  const bool vec2 = s->dtype == DSV_C64 && !(mask & 1ull) && s->nbits >= 1;
  const int sh = vec2 ? 1 : 0;
  ProfTok t = prof_start(s);
  CKL(launch_collapse(s->dtype, vec2 ? MODE_VEC2 : MODE_SCALAR, namps(s) >> sh, mask >> sh, val >> sh,
                      1.0 / std::sqrt(norm2_kept), s->d, s->stream), 1);
  prof_stop(s, t, PC_COLLAPSE, 2.0 * double(amp_bytes(s->dtype)) * double(namps(s)));
  return DSV_OK;
}

int dsv_scale(dsv_state* s, double factor) {
  if (int rc = check_state(s)) return rc;
  DeviceGuard g(s->device);
  const bool vec2 = s->dtype == DSV_C64 && s->nbits >= 1;
  const int sh = vec2 ? 1 : 0;
  ProfTok t = prof_start(s);
  CKL(launch_collapse(s->dtype, vec2 ? MODE_VEC2 : MODE_SCALAR, namps(s) >> sh, 0, 0, factor, s->d, s->stream), 1);
  prof_stop(s, t, PC_COLLAPSE, 2.0 * double(amp_bytes(s->dtype)) * double(namps(s)));
  return DSV_OK;
}

int dsv_sample(dsv_state* s, const double* variates, int64_t shots, uint64_t* outcomes) {
  if (int rc = no_capture(s, "dsv_sample")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(s)) return rc;
  if (shots < 1) return fail(DSV_EINVAL, "shots must be >= 1");
  DeviceGuard g(s->device);
  // 1) ordered chunk sums of |a|^2 over kChunk-amplitude chunks (scalar units)
  double* d_partial = nullptr;
  uint64_t nch = 0;
  uint64_t chunk_amps = uint64_t(kReduceThreads) * kReduceUnitsPerThread;  // scalar-unit fallback
  if (int rc = probs_impl(s, nullptr, 0, false, nullptr, &d_partial, &nch, &chunk_amps)) return rc;
  std::vector<double> cs(nch);
  CK(cudaMemcpyAsync(cs.data(), d_partial, sizeof(double) * nch, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  // 2) host prefix over chunks (sequential, float64)
  std::vector<double> pre(nch);
  double run = 0.0;
  for (uint64_t c = 0; c < nch; ++c) {
    run += cs[c];
    pre[c] = run;
  }
  const double total = run;
  if (!(total > 0.0)) return fail(DSV_EINVAL, "state has zero norm; cannot sample");
  std::vector<uint64_t> ch(shots);
  std::vector<double> rs(shots);
  for (int64_t i = 0; i < shots; ++i) {
    const double target = variates[i] * total;
    uint64_t c = uint64_t(std::upper_bound(pre.begin(), pre.end(), target) - pre.begin());
    if (c >= nch) c = nch - 1;
    ch[i] = c;
    rs[i] = target - (c ? pre[c - 1] : 0.0);
  }
  // 3) per-shot warp scan inside the chunk
  const size_t b1 = ((sizeof(uint64_t) * shots + 255) / 256) * 256;
  const size_t need = 3 * b1;
  if (int rc = ensure_scratch(s, need)) return rc;
  char* base = static_cast<char*>(s->scratch);
  uint64_t* d_ch = reinterpret_cast<uint64_t*>(base);
  double* d_rs = reinterpret_cast<double*>(base + b1);
  uint64_t* d_out = reinterpret_cast<uint64_t*>(base + 2 * b1);
  CK(cudaMemcpyAsync(d_ch, ch.data(), sizeof(uint64_t) * shots, cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemcpyAsync(d_rs, rs.data(), sizeof(double) * shots, cudaMemcpyHostToDevice, s->stream));
  ProfTok t = prof_start(s);
  CKL(launch_sample_scan(s->dtype, namps(s), chunk_amps, shots, d_ch, d_rs, s->d, d_out, s->stream), 1);
  prof_stop(s, t, PC_SAMPLE, double(amp_bytes(s->dtype)) * double(chunk_amps) * double(shots));
  CK(cudaMemcpyAsync(outcomes, d_out, sizeof(uint64_t) * shots, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return DSV_OK;
}

// ---- segments -----------------------------------------------------------------------------

int dsv_exchange_halves(dsv_state* a, dsv_state* b, int local_bit, int part, int nparts) {
  if (int rc = no_capture(a, "dsv_exchange_halves")) return rc;
  if (int rc = no_capture(b, "dsv_exchange_halves")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(a)) return rc;
  if (int rc = check_state(b)) return rc;
  if (a->nbits != b->nbits || a->dtype != b->dtype) return fail(DSV_EINVAL, "exchange between segments of different shape");
  if (local_bit < 0 || local_bit >= a->nbits) return fail(DSV_EINVAL, "local bit %d out of range", local_bit);
  if (nparts < 1 || part < 0 || part >= nparts) return fail(DSV_EINVAL, "bad exchange slice %d/%d", part, nparts);
  DeviceGuard g(a->device);
  if (!b->ipc && a->device != b->device)
    if (int rc = enable_peer(a->device, b->device)) return rc;
  if (!b->ipc)
    if (int rc = sync_streams(a, b)) return rc;
  const bool vec2 = a->dtype == DSV_C64 && local_bit != 0;
  const int sh = vec2 ? 1 : 0;
  const uint64_t T = namps(a) >> (1 + sh);
  const uint64_t lo = T / nparts * part + std::min<uint64_t>(part, T % nparts);
  const uint64_t hi = lo + T / nparts + (uint64_t(part) < T % nparts ? 1 : 0);
  ProfTok t = prof_start(a);
  CKL(launch_exchange_halves(a->dtype, vec2 ? MODE_VEC2 : MODE_SCALAR, local_bit - sh, lo, hi, a->d, b->d, a->stream), 1);
  prof_stop(a, t, PC_EXCHANGE, 4.0 * double(amp_bytes(a->dtype)) * double(hi - lo) * (vec2 ? 2.0 : 1.0));
  if (!b->ipc)
    if (int rc = sync_streams(b, a)) return rc;
  return DSV_OK;
}

int dsv_exchange_all(dsv_state* a, dsv_state* b) {
  if (int rc = no_capture(a, "dsv_exchange_all")) return rc;
  if (int rc = no_capture(b, "dsv_exchange_all")) return rc;
  DSV_NVTX_RANGE();
  if (int rc = check_state(a)) return rc;
  if (int rc = check_state(b)) return rc;
  if (a->nbits != b->nbits || a->dtype != b->dtype) return fail(DSV_EINVAL, "exchange between segments of different shape");
  DeviceGuard g(a->device);
  if (!b->ipc && a->device != b->device)
    if (int rc = enable_peer(a->device, b->device)) return rc;
  if (!b->ipc)
    if (int rc = sync_streams(a, b)) return rc;
  ProfTok t = prof_start(a);
  CKL(launch_exchange_all(a->dtype, namps(a), a->d, b->d, a->stream), 1);
  prof_stop(a, t, PC_EXCHANGE, 4.0 * double(amp_bytes(a->dtype)) * double(namps(a)));
  if (!b->ipc)
    if (int rc = sync_streams(b, a)) return rc;
  return DSV_OK;
}

// ---- masked exchange (batched (global, local) swaps) ----------------------------------

namespace {

struct MaskedPlan {
  Geom g;
  int mode = MODE_SCALAR;
  uint64_t pa = 0, pb = 0;
  int la = 0, lb = 0;
};

int plan_masked(const dsv_state* a, const dsv_state* b, const int32_t* lbits, int q, uint64_t pat_a,
                uint64_t pat_b, MaskedPlan* mp) {
  if (int rc = check_state(a)) return rc;
  if (int rc = check_state(b)) return rc;
  if (a->nbits != b->nbits || a->dtype != b->dtype) return fail(DSV_EINVAL, "exchange between segments of different shape");
  if (q < 1 || q > 8 || !lbits) return fail(DSV_EINVAL, "masked exchange over %d bits", q);
  uint64_t mask = 0;
  for (int i = 0; i < q; ++i) {
    const int l = lbits[i];
    if (l < 0 || l >= a->nbits) return fail(DSV_EINVAL, "local bit %d out of range", l);
    if (mask >> l & 1) return fail(DSV_EINVAL, "local bits must be distinct");
    mask |= 1ull << l;
  }
  if ((pat_a | pat_b) & ~mask) return fail(DSV_EINVAL, "exchange patterns outside the local bits");
  std::vector<int> holes;
  if (a->dtype == DSV_C128) {
    mp->mode = MODE_SCALAR;
    for (int b2 = 0; b2 < 64; ++b2)
      if (mask >> b2 & 1) holes.push_back(b2);
    mp->pa = pat_a;
    mp->pb = pat_b;
    return make_geom(a->nbits, holes, 0, &mp->g);
  }
  // complex64: 16-byte units of amplitude pairs; bit 0 among the local bits -> lane mode
  mp->mode = (mask & 1) ? MODE_SCALAR : MODE_VEC2;
  mp->la = int(pat_a & 1);
  mp->lb = int(pat_b & 1);
  for (int b2 = 1; b2 < 64; ++b2)
    if (mask >> b2 & 1) holes.push_back(b2 - 1);
  mp->pa = pat_a >> 1;
  mp->pb = pat_b >> 1;
  return make_geom(a->nbits - 1, holes, 0, &mp->g);
}

// slice [part/nparts] of the masked exchange, launched on `run`'s stream / device
int run_masked(dsv_state* run, dsv_state* a, dsv_state* b, const MaskedPlan& mp, int part, int nparts) {
  const uint64_t T = mp.g.nwork;
  const uint64_t lo = T / nparts * part + std::min<uint64_t>(part, T % nparts);
  const uint64_t hi = lo + T / nparts + (uint64_t(part) < T % nparts ? 1 : 0);
  ProfTok t = prof_start(run);
  CKL(launch_exchange_masked(a->dtype, mp.mode, mp.g, mp.pa, mp.pb, mp.la, mp.lb, lo, hi, a->d, b->d, run->stream), 1);
  // bytes: every 16-byte unit of the slice read and written on both sides
  prof_stop(run, t, PC_EXCHANGE, 4.0 * 16.0 * double(hi - lo));
  return DSV_OK;
}

}  // namespace

int dsv_exchange_masked(dsv_state* a, dsv_state* b, const int32_t* lbits, int q, uint64_t pat_a, uint64_t pat_b,
                        int part, int nparts) {
  if (int rc = no_capture(a, "dsv_exchange_masked")) return rc;
  if (int rc = no_capture(b, "dsv_exchange_masked")) return rc;
  DSV_NVTX_RANGE();
  MaskedPlan mp;
  if (int rc = plan_masked(a, b, lbits, q, pat_a, pat_b, &mp)) return rc;
  if (nparts < 1 || part < 0 || part >= nparts) return fail(DSV_EINVAL, "bad exchange slice %d/%d", part, nparts);
  DeviceGuard g(a->device);
  if (!b->ipc && a->device != b->device)
    if (int rc = enable_peer(a->device, b->device)) return rc;
  if (!b->ipc)
    if (int rc = sync_streams(a, b)) return rc;
  if (int rc = run_masked(a, a, b, mp, part, nparts)) return rc;
  if (!b->ipc)
    if (int rc = sync_streams(b, a)) return rc;
  return DSV_OK;
}

int dsv_exchange_pair(dsv_state* a, dsv_state* b, const int32_t* lbits, int q, uint64_t pat_a, uint64_t pat_b) {
  if (int rc = no_capture(a, "dsv_exchange_pair")) return rc;
  if (int rc = no_capture(b, "dsv_exchange_pair")) return rc;
  DSV_NVTX_RANGE();
  MaskedPlan mp;
  if (int rc = plan_masked(a, b, lbits, q, pat_a, pat_b, &mp)) return rc;
  if (a->ipc || b->ipc) return fail(DSV_EINVAL, "dsv_exchange_pair needs two local segments (use dsv_exchange_masked)");
  if (a->device != b->device) {
    if (int rc = enable_peer(a->device, b->device)) return rc;
    if (int rc = enable_peer(b->device, a->device)) return rc;
  }
  {
    DeviceGuard g(a->device);
    if (int rc = sync_streams(a, b)) return rc;
  }
  {
    DeviceGuard g(b->device);
    if (int rc = sync_streams(b, a)) return rc;
  }
  {
    DeviceGuard g(a->device);
    if (int rc = run_masked(a, a, b, mp, 0, 2)) return rc;
  }
  {
    DeviceGuard g(b->device);
    if (int rc = run_masked(b, a, b, mp, 1, 2)) return rc;
  }
  {
    DeviceGuard g(a->device);
    if (int rc = sync_streams(a, b)) return rc;
  }
  {
    DeviceGuard g(b->device);
    if (int rc = sync_streams(b, a)) return rc;
  }
  return DSV_OK;
}

int dsv_stream_join(dsv_state* waiter, dsv_state* other) {
  if (int rc = check_state(waiter)) return rc;
  if (int rc = check_state(other)) return rc;
  if (waiter->ipc || other->ipc) return fail(DSV_EINVAL, "stream join of a peer mapping");
  DeviceGuard g(waiter->device);
  return sync_streams(waiter, other);
}

// ---- group reductions: one launch per segment, all devices concurrently ---------------------

extern "C++" {
namespace {

template <class F>
int group_reduce(dsv_state** s, int count, size_t per, double* out, F&& op) {
  if (!s || count < 1 || !out) return fail(DSV_EINVAL, "empty segment group");
  for (int i = 0; i < count; ++i)
    if (int rc = check_state(s[i])) return rc;
  int rc = DSV_OK;
  int issued = 0;
  for (; issued < count; ++issued) {
    dsv_state* st = s[issued];
    st->defer = true;
    st->pending_n = 0;
    rc = op(st);
    st->defer = false;
    if (rc) break;
  }
  for (int i = 0; i < issued; ++i) {
    DeviceGuard g(s[i]->device);
    cudaError_t e = cudaStreamSynchronize(s[i]->stream);
    if (e != cudaSuccess && !rc) rc = cuda_fail(e, "cudaStreamSynchronize");
    if (!rc) {
      if (s[i]->pending_n != per) rc = fail(DSV_EINVAL, "reduction produced %zu values, expected %zu", s[i]->pending_n, per);
      else std::memcpy(out + per * size_t(i), s[i]->pinned, sizeof(double) * per);
    }
  }
  return rc;
}

}  // namespace
}  // extern "C++"

int dsv_group_norm2(dsv_state** s, int count, double* out) {
  return group_reduce(s, count, 1, out, [](dsv_state* st) { return dsv_norm2(st, nullptr); });
}

int dsv_group_marginal_probs(dsv_state** s, int count, const int32_t* bits, int k, double* out) {
  if (k < 0 || k > 26) return fail(DSV_EUNSUPPORTED, "marginal over %d bits not supported (max 26)", k);
  return group_reduce(s, count, size_t(1) << k, out,
                      [&](dsv_state* st) { return dsv_marginal_probs(st, bits, k, nullptr); });
}

int dsv_group_expect_pauli(dsv_state** s, int count, const int32_t* bits, const char* paulis, int m, double* out) {
  return group_reduce(s, count, 2, out, [&](dsv_state* st) { return dsv_expect_pauli(st, bits, paulis, m, nullptr); });
}

// ---- CUDA graphs: record a gate sequence once, replay it -------------------------------------

struct dsv_graph {
  dsv_state* state = nullptr;
  int device = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<void*> bufs;  // per-gate tables baked at capture time
};

int dsv_capture_begin(dsv_state* s) {
  if (int rc = check_state(s)) return rc;
  if (s->capturing) return fail(DSV_EINVAL, "already capturing");
  if (s->ipc) return fail(DSV_EINVAL, "cannot capture on a peer mapping");
  DeviceGuard g(s->device);
  s->keep_gdata = s->gdata;
  s->keep_gdata_bytes = s->gdata_bytes;
  s->keep_scratch = s->scratch;
  s->keep_scratch_bytes = s->scratch_bytes;
  s->cap_bufs.clear();
  CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeRelaxed));
  s->capturing = true;
  return DSV_OK;
}

static void capture_restore(dsv_state* s) {
  s->capturing = false;
  s->gdata = s->keep_gdata;
  s->gdata_bytes = s->keep_gdata_bytes;
  s->scratch = s->keep_scratch;
  s->scratch_bytes = s->keep_scratch_bytes;
}

int dsv_capture_end(dsv_state* s, dsv_graph** out) {
  if (int rc = check_state(s)) return rc;
  if (!out) return fail(DSV_EINVAL, "null argument");
  *out = nullptr;
  if (!s->capturing) return fail(DSV_EINVAL, "not capturing");
  DeviceGuard g(s->device);
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(s->stream, &graph);
  capture_restore(s);
  dsv_graph* gr = new dsv_graph;
  gr->state = s;
  gr->device = s->device;
  gr->bufs.swap(s->cap_bufs);
  if (e != cudaSuccess) {
    dsv_graph_destroy(gr);
    return cuda_fail(e, "cudaStreamEndCapture");
  }
  gr->graph = graph;
  const cudaError_t e2 = cudaGraphInstantiate(&gr->exec, graph, 0);
  if (e2 != cudaSuccess) {
    dsv_graph_destroy(gr);
    return cuda_fail(e2, "cudaGraphInstantiate");
  }
  *out = gr;
  return DSV_OK;
}

int dsv_graph_launch(dsv_graph* g, dsv_state* s) {
  if (!g || !g->exec) return fail(DSV_EINVAL, "null graph");
  if (int rc = check_state(s)) return rc;
  if (g->state != s) return fail(DSV_EINVAL, "a graph replays on the state it was captured on");
  if (int rc = no_capture(s, "dsv_graph_launch")) return rc;
  DeviceGuard dg(s->device);
  CKL(cudaGraphLaunch(g->exec, s->stream), 1);
  return DSV_OK;
}

int dsv_graph_destroy(dsv_graph* g) {
  if (!g) return DSV_OK;
  DeviceGuard dg(g->device);
  cudaDeviceSynchronize();  // a replay may still be reading the baked tables
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  for (void* p : g->bufs) cudaFree(p);
  delete g;
  return DSV_OK;
}

int dsv_ipc_handle(dsv_state* s, void* out64) {
  if (int rc = check_state(s)) return rc;
  if (s->ipc) return fail(DSV_EINVAL, "cannot re-export a peer mapping");
  DeviceGuard g(s->device);
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, s->d));
  s->exported = true;
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(out64, &h, 64);
  return DSV_OK;
}

int dsv_peer_open(int device, int nbits, int dtype, const void* handle64, dsv_state** out) {
  if (!out || !handle64) return fail(DSV_EINVAL, "null argument");
  *out = nullptr;
  DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  dsv_state* s = new dsv_state;
  s->device = device;
  s->nbits = nbits;
  s->dtype = dtype;
  s->owned = false;
  s->ipc = true;
  cudaError_t e = cudaIpcOpenMemHandle(&s->d, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    delete s;
    return cuda_fail(e, "cudaIpcOpenMemHandle");
  }
  e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    cudaIpcCloseMemHandle(s->d);
    delete s;
    return cuda_fail(e, "cudaStreamCreate");
  }
  *out = s;
  return DSV_OK;
}

// ---- instrumentation ---------------------------------------------------------------------

int dsv_prof_enable(dsv_state* s, int on) {
  if (int rc = check_state(s)) return rc;
  s->prof_on = on != 0;
  return DSV_OK;
}

int dsv_prof_reset(dsv_state* s) {
  if (int rc = check_state(s)) return rc;
  DeviceGuard g(s->device);
  CK(cudaStreamSynchronize(s->stream));
  for (auto& r : s->recs) {
    s->ev_pool.push_back(r.a);
    s->ev_pool.push_back(r.b);
  }
  s->recs.clear();
  return DSV_OK;
}

int dsv_prof_read(dsv_state* s, uint64_t* count, double* ms, double* bytes) {
  if (int rc = check_state(s)) return rc;
  DeviceGuard g(s->device);
  CK(cudaStreamSynchronize(s->stream));
  for (int c = 0; c < DSV_PROF_NCLASS; ++c) {
    count[c] = 0;
    ms[c] = 0.0;
    bytes[c] = 0.0;
  }
  for (auto& r : s->recs) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    count[r.cls] += 1;
    ms[r.cls] += t;
    bytes[r.cls] += r.bytes;
  }
  return DSV_OK;
}

const char* dsv_prof_class_name(int c) {
  if (c < 0 || c >= DSV_PROF_NCLASS) return "";
  return kProfNames[c];
}

int dsv_event_record(dsv_state* s, int slot) {
  if (int rc = check_state(s)) return rc;
  if (slot < 0 || slot >= 16) return fail(DSV_EINVAL, "event slot out of range");
  DeviceGuard g(s->device);
  if (!s->uev[slot]) CK(cudaEventCreate(&s->uev[slot]));
  CK(cudaEventRecord(s->uev[slot], s->stream));
  return DSV_OK;
}

int dsv_event_elapsed(dsv_state* s, int a, int b, float* ms) {
  if (int rc = check_state(s)) return rc;
  if (a < 0 || a >= 16 || b < 0 || b >= 16 || !s->uev[a] || !s->uev[b]) return fail(DSV_EINVAL, "event slot not recorded");
  DeviceGuard g(s->device);
  CK(cudaEventSynchronize(s->uev[b]));
  CK(cudaEventElapsedTime(ms, s->uev[a], s->uev[b]));
  return DSV_OK;
}

}  // extern "C"
