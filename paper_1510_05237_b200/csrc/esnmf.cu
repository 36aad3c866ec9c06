// esnmf.cu -- libesnmf.so: C ABI (include/esnmf.h) and host orchestration of
// the enforced-sparse ALS hot path on one B200 (sm_100a) per process.
//
// Per iteration (Alg. 2; per-column enforcement P:304):
//   V side:  G_U = U^T U -> W = (G_U + eps I)^{-1} (k_sweep_regs) -> Z = U W
//            -> LS_V = A^T Z: tail terms by row gather (k_spmm_tail), the most
//               frequent terms on tcgen05 (k_vhead_otf, which also merges the
//               tail rows); kpad <= 8: a narrow SpMM (k_spmm_narrow)
//            -> clamp + top-t per column (k_select.cuh) -> V
//   U side:  G_V, W on a second stream beside Y = A V (fixed-point scatter from
//            the active documents, k_uside_scatter) -> LS_U = Y W (k_uside_tc on
//            tcgen05, or the fp32/fp64 SIMT finish) -> clamp + top-t -> U
//   R (direct difference) and E (trace identity), launched at the
//   start of the next iteration on the second stream.
// Steady-state iterations are replayed as CUDA graphs; the host never
// synchronises inside esnmf_iterate.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/esnmf.h"
#include "common.cuh"
#include "k_csr.cuh"
#include "k_factor.cuh"
#include "k_merge.cuh"
#include "k_metrics.cuh"
#include "k_select.cuh"
#include "k_solve.cuh"
#include "k_spmm_terms.cuh"
#include "k_uside_scatter.cuh"
#include "k_vhead.cuh"
#include "k_uside_tc.cuh"
#include "k_spmm_tail.cuh"
#include "k_vtail.cuh"
#include "k_seq.cuh"

using namespace esk;

namespace {

thread_local std::string g_last_error;

struct Fail {
  esnmf_status st;
};

[[noreturn]] void fail(esnmf_status st, const std::string& msg) {
  g_last_error = msg;
  throw Fail{st};
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) fail(ESNMF_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    fail(ESNMF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define CK(x) ck((x), #x)
#define CKL(name) ck(cudaGetLastError(), name)

constexpr int64_t kSplitLen = 4096;  // max stored entries per SpMM work item (A rows)
constexpr int kMaxGramSeg = 64;        // sparse Gram: entry segments per column
constexpr int kMaxGramSegDense = 296;  // dense Gram: row slabs (2 per SM)
constexpr int64_t kSelScanMax = 4096;  // flat selection: segment-scan blocks (k * rows < 2^31 needs < 1024)

struct DevCsr {
  int64_t rows = 0, cols = 0, nnz = 0;
  int64_t* ptr = nullptr;
  int2* ent = nullptr;
  RowChunk* chunks = nullptr;  // balanced work units (create-time passes)
  int64_t nchunks = 0;
};

struct Factor {
  int64_t rows = 0, cap = 0, cap_rows = 0;
  int64_t* colptr = nullptr;
  int32_t* row = nullptr;
  float* val = nullptr;
  int32_t* rowmap = nullptr;
  int32_t* active = nullptr;
  int64_t* n_active = nullptr;
  float* dense = nullptr;
  int64_t maxcol = 0;  // host upper bound of a column's length
  bool has = false;
};

struct Side {
  int64_t row0 = 0, rows = 0, ldx = 0;  // this rank's output rows
  float* X = nullptr;                   // LS, column-major k x ldx
  float* Xt = nullptr;                  // V side with a head: tail part, row-major rows x kpad
  DevCsr T;                             // operator rows of this shard (local row ids)
  // work items (U side only)
  WorkItem* items = nullptr;
  int32_t* item_slot = nullptr;
  int64_t nitems = 0;
  SplitRow* splits = nullptr;
  int64_t nsplit = 0, nslots = 0;
  float* partial = nullptr;
  // selection scratch
  int64_t nchunks = 0;
  uint32_t* hist = nullptr;
  ColSel* sel = nullptr;
  uint64_t* cand = nullptr;
  int32_t* cand_fill = nullptr;
  int64_t* chunk_cnt = nullptr;
  int64_t* coltot = nullptr;
  uint64_t* kthr = nullptr;
  SelLvl* lvl = nullptr;          // [k] multi-block radix fallback state
  int64_t* scanbuf = nullptr;     // [kSelScanMax] block sums of the flat view's segment scan
  int ccap = 0;                   // candidate list capacity per column (cand)
  uint64_t* above = nullptr;      // two-pass select (t <= kSelFastT): [k][t] row keys
  int64_t above_t = -1;           // its t capacity per column
  int32_t* above_fill = nullptr;  // [k] (followed by bucket_fill [k] in the same allocation)
  uint64_t* bucket = nullptr;     // [k][kSelCap] value keys of the threshold bucket
  // predicted-threshold candidates (the previous select's t-th value - 10 %)
  uint32_t* pred = nullptr;       // [k] value bits; 0xFFFFFFFF = no prediction
  uint64_t* pcand = nullptr;      // [k][pcap]
  int32_t* pfill = nullptr;       // [k] then done [k]
  int pcap = 0;
  int32_t* npos = nullptr;        // [k] positives per column (fused V-side pass 1)
  bool fused = false;             // this half-step's pass 1 ran in the head epilogue
  bool xdeferred = false;         // ... and the head did not write X (written only if a prediction fails)
  bool ls_stored = true;          // X holds this side's last LS (esnmf_get_ls)
  int* xneed = nullptr;           // [1] device: some column's prediction failed (gates the head re-run)
  // Gram of the factor this side reads, and its eps
  double* G = nullptr;
  double* eps = nullptr;
  int64_t* peak = nullptr;  // positives of the clamped LS of the last select (record peak nnz)
  bool ls_valid = false;
  // multi-rank: local top-t, exchange buffers, merge scratch (k_merge.cuh)
  int64_t cap_s = 0;            // candidates per column per rank
  int64_t* lcolptr = nullptr;
  int32_t* lrow = nullptr;
  float* lval = nullptr;
  void* sendbuf = nullptr;
  void* recvbuf = nullptr;
  size_t shard_bytes = 0;
  uint64_t* mscratch = nullptr;
};

// ---- built-in NCCL collectives (esnmf_nccl_*; libnccl.so.2 loaded at run time) ----
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      a.error = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(lib, "ncclCommInitRank"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(lib, "ncclAllGather"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(lib, "ncclAllReduce"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(lib, "ncclCommDestroy"));
    a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(lib, "ncclGetErrorString"));
    if (!a.getUniqueId || !a.commInitRank || !a.allGather || !a.allReduce || !a.commDestroy || !a.getErrorString)
      a.error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

struct NcclCtx {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
};

int nccl_allgather_cb(void* ctx, const void* send, void* recv, int64_t bytes, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  return nccl_api().allGather(send, recv, (size_t)bytes, ncclUint8, c->comm, (cudaStream_t)stream) == ncclSuccess ? 0
                                                                                                               : 1;
}

int nccl_allreduce_cb(void* ctx, double* buf, int64_t count, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  return nccl_api().allReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, c->comm, (cudaStream_t)stream) ==
                 ncclSuccess
             ? 0
             : 1;
}

// a communicator the library owns: stream-ordered device collectives, CUDA-graph capturable
bool builtin_nccl(const esnmf_comm& c) { return c.allgather == nccl_allgather_cb && c.allreduce_sum_f64 == nccl_allreduce_cb; }

}  // namespace

struct esnmf {
  int dev = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // second stream for work that overlaps the main chain (fork/join by events):
  // the U side's Gram + solve run beside the active-document scatter, and the
  // error/record kernels of iteration i beside the V side of iteration i+1
  cudaStream_t aux = nullptr;
  // the previous iteration's record kernels (R, E; a7, a8): lowest priority, so
  // the solves queued on aux are scheduled first when the V side's tail starts
  cudaStream_t maux = nullptr;
  cudaEvent_t ev_ufork = nullptr, ev_ujoin = nullptr, ev_mfork = nullptr, ev_mjoin = nullptr;
  bool aux_pending = false;
  bool u_prefork = false;        // the U side's Gram + solve already enqueued on aux (after V's row view)
  int64_t n = 0, m = 0, nnz = 0;
  int k = 0, kpad = 0;
  int64_t t = 0;  // < 0 unlimited (create's t)
  int64_t tside[2] = {0, 0};  // budgets per side: [0] t_v (V side), [1] t_u (U side)
  bool whole = false;         // whole-factor enforcement (Alg. 2 as printed)
  int64_t init_nnz = 0;       // > 0: sparse U_0 (reading C18)
  // sequential ALS (Alg. 3, k_seq.cuh): the pipeline above runs on the current
  // block of k = seq_k2 columns; the ktot - k converged columns are in FU / FV
  int ktot = 0, kpf = 0;       // all topics and their row stride (0: not sequential)
  int seq_k2 = 0, seq_iters = 0, seq_b = 0, seq_i = 0;
  Factor FU, FV;               // U_1, V_1: columns [0, seq_b k2) of ktot
  double* seqC = nullptr;      // [ktot][k2] H_1^T H_2
  double* seqM = nullptr;      // [ktot][k2] (H_1^T H_2) W_22
  double* seqc = nullptr;      // [3] T_1, S_11, ||U_1||^2 (record constants of the block)
  int64_t* wcolptr = nullptr; // [2] colptr of the flat (one-column) selection
  double rho = 1e-10;
  uint64_t seed = 0;
  int world = 1, rank = 0;
  bool sharded = false;        // the multi-rank paths (world > 1; or ESNMF_FORCE_SHARDED=1 with a comm, tests)
  esnmf_comm comm{};
  Side side[2];  // 0: V side (A^T rows = documents), 1: U side (A rows = terms)
  Factor U[2];
  int ucur = 0;
  Factor V;
  float* Z = nullptr;
  float* zc = nullptr;          // kpad <= 8: compact term-indexed z = U W, kpad per term (k_spmm_narrow)
  int zs = 0;                   // V-side Z row stride (floats), term-indexed rows
  int32_t* zlist = nullptr;     // terms whose Z rows were written last
  int64_t* zcount = nullptr;
  uint32_t* tbits = nullptr;    // active-term bitmap of U
  double* W = nullptr;
  double* gram_partial = nullptr;
  double* sweep_scratch = nullptr;
  // row-CSR of V for the U side
  uint32_t* vbits = nullptr;  // [ceil(m/32)]
  uint64_t* vmap = nullptr;   // [m]
  int2* vent = nullptr;       // [V.cap]
  int64_t* vrptr = nullptr;   // [V.cap_rows + 1]
  int64_t* vcur = nullptr;    // [V.cap_rows + 1]
  int64_t* vscan = nullptr;   // scan block sums
  uint32_t* vmax = nullptr;   // bits of max(V) (fixed-point scale of the U side)
  double* rsum = nullptr;     // [n_local] row sums of A (fixed-point scale of the U side)
  double* rsum_max = nullptr; // max_i rsum[i]
  unsigned long long* Yq = nullptr;  // [n][kpad] fixed-point A V (single-GPU U side): Yqb[ucur] during a U side
  unsigned long long* Yqb[2] = {nullptr, nullptr};  // double buffer: k_polish_u reads Yq after the select;
                                                    // the next V side clears it (aux stream)
  bool v_since_u = true;             // a V side ran since the last U side (Yqb[yq_par] is clear)
  int yq_par = 0;                    // the buffer the next U side uses (flips every U side)
  bool yq_other_dirty = false;       // Yqb[1 - yq_par] (the last U side's) still holds its sums
  float* W32 = nullptr;              // [k][kpad] fp32 copy of W for k_uside_finish_rt
  uint8_t* wtc = nullptr;            // W as the tensor-core B operand (fp16 hi/lo, k_uside_tc)
  float* wtc_scale = nullptr;        // [kn] its per-column scales
  int utc_kn = 0, utc_kk = 0;        // 0: k_uside_tc not used (kpad > 128)
  // V-side tensor-core head (k_vhead.cuh): h most frequent terms, dense fp16 hi/lo tiles
  int head_h = 0, head_nchunks = 0, kn = 0, head_acc_cols = 0;
  bool keep_ls = false;   // esnmf_options.keep_ls: every V side writes its LS buffer
  bool force_ls = false;  // esnmf_half_step in progress: write it
  int64_t head_ntiles = 0;
  int32_t* headterm = nullptr;   // [h] term of head slot s
  int32_t* headslot = nullptr;   // [n] head slot of term i, -1 if not in the head
  uint8_t* zhead = nullptr;      // [chunks][kn x 64 x 2 x 2 B] Z head rows, hi/lo
  float* colscale = nullptr;     // [kn] 2^-(eA + eZ_c)
  unsigned* amax_bits = nullptr; // max value of this rank's A^T shard (float bits)
  int32_t* nh = nullptr;         // [v rows] head entries at the front of each A^T row
  int head_nd = 0;               // leading head chunks stored as dense tiles (atile)
  uint8_t* atile = nullptr;      // [tiles][nd][32 KB] dense fp16 hi/lo tiles of those chunks
  int64_t* hoff = nullptr;       // [tiles * sparse chunks + 1] segment offsets of the tiled head copy
  int2* hseg = nullptr;          // head entries by (tile, chunk): (row in tile << 6 | slot, value)
  // V-side tail in the paper's order (k_vtail.cuh): A^T_tail U per tile, then
  // (Y_tail W) as nyc extra K-chunks of the head kernel; off: the Z-row gather
  bool ptail = false;
  int nyc = 0;
  int64_t* toff = nullptr;       // [tiles + 1] tail entries of each tile (jagged-diagonal order)
  int2* tent = nullptr;          // (row in tile << 24 | term, value)
  uint8_t* ytile = nullptr;      // [tiles][128 x kn x 4 B] Y_tail as fp16 hi/lo chunks
  uint8_t* wbuf = nullptr;       // [nyc][kn x 64 x 4 B] W' as the B operand
  unsigned* rowsum_bits = nullptr;  // max document row sum of A^T (float bits, rounded up; global)
  uint64_t* umap = nullptr;      // [n] U row view: (first << 32) | count
  uint32_t* ubits = nullptr;     // [n / 32] rows of U with a nonzero
  double* Z64 = nullptr;         // [n terms][k] Z = U W in fp64 for U's active rows (k_form_z64); others stale
  double vt_kmax = 1e4, vt_amax = 8.0;  // k_vcond_flag thresholds (ESNMF_VT_KMAX / ESNMF_VT_AMAX)
  double vt_ratio = 8.0;         // cost of a paper-order product / a gathered FMA (ESNMF_VT_RATIO)
  int32_t* termlen = nullptr;    // [n] stored entries of each term (row lengths of A, global)
  double* vcost = nullptr;       // [8] the last V side's cost model (k_urows_finish)
  unsigned* vt_ticket = nullptr; // [1] k_urows_finish's last-block ticket (zero between launches)
  bool polish = true;            // kept V values recomputed exactly (ESNMF_NO_POLISH=1: off)
  double u_kmax = 100.0;         // U side: (Y W) in fp32 / fp16 hi/lo only for kappa_inf <= this (ESNMF_U_KMAX)
  unsigned long long* vt_next = nullptr;  // k_ytail's tile counter
  int2* uent = nullptr;          // [U cap] (column, value * 2^s_c)
  int64_t* urptr = nullptr;      // [U cap_rows + 1]
  int64_t* ucursor = nullptr;
  int64_t* uscan = nullptr;
  int32_t* ulist = nullptr;      // rows published in umap (cleared before the next build)
  int64_t* ulist_n = nullptr;
  uint32_t* umax = nullptr;      // [k] max of U over the tail rows, per column (float bits)
  int* ushift = nullptr;         // [k] fixed-point exponents s_c
  uint32_t* gmax_buf = nullptr;  // multi-rank: allgather of {amax, rowsum} (16 B per rank)
  cudaEvent_t ev_vfork = nullptr, ev_vjoin = nullptr;
  cudaEvent_t ev_ugram = nullptr;  // the U side's Gram done on aux (the scatter waits on it)
  cudaEvent_t ev_gfork = nullptr, ev_gjoin = nullptr;  // the record's Gram of U on aux
  bool gram_on_aux = false;  // G_U was last computed on aux (a main-stream reader joins first)
  int64_t u_rows_max = 0, v_rows_max = 0;  // largest shard over ranks
  int num_sms = 148;
  int smem_optin = 227 * 1024;
  int* flags = nullptr;  // [0] singular, [1] validation, [2] U0 invalid
  double* red = nullptr;
  int64_t red_cap = 0;
  double* scal = nullptr;
  double* normA2_dev = nullptr;
  esnmf_record* rec = nullptr;
  int64_t rec_cap = 0, nrec = 0;
  int64_t* d_nrec = nullptr;   // device mirror of nrec: k_finalize_record's slot (graph replays)
  // CUDA graphs of two steady-state iterations (one per parity of ucur), replayed
  // by esnmf_iterate; any other state change drops them (graph_reset)
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  esnmf_record* grec[2] = {nullptr, nullptr};
  int64_t glaunch[2] = {0, 0};
  int steady = 0;              // eager iterations since the last state change
  bool metrics_pending = false;  // the last iteration's record is not launched yet (flush_metrics)
  double normA2 = 0;
  bool gramU_valid = false;
  int64_t nlaunch = 0;  // kernels enqueued by this handle (esnmf_get_info)
  // per-phase CUDA-event profiling (esnmf_profile / esnmf_phase_times)
  bool prof_on = false;
  struct ProfRec {
    int id;
    cudaEvent_t a, b;
  };
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[16] = {0};
  int64_t prof_calls[16] = {0};
  std::vector<void*> allocs;
  int64_t bytes = 0;
  double alloc_ms = 0;  // host time spent in cudaMalloc (ESNMF_CREATE_TIMING)

  // Device buffers come from a library-owned stream-ordered memory pool per device
  // (release threshold: never; trimmed to 24 GB when a handle is destroyed), so the
  // next esnmf_create reuses a destroyed handle's pages instead of mapping fresh ones
  // (cudaMalloc of ~130 buffers took 17-90 ms per create).  ESNMF_NO_POOL=1: cudaMalloc.
  cudaMemPool_t pool = nullptr;
  template <typename T>
  T* alloc(int64_t count) {
    if (count <= 0) count = 1;
    void* p = nullptr;
    size_t b = sizeof(T) * (size_t)count;
    const auto t0 = std::chrono::steady_clock::now();
    if (pool) ck(cudaMallocFromPoolAsync(&p, b, pool, stream), "cudaMallocFromPoolAsync");
    else ck(cudaMalloc(&p, b), "cudaMalloc");
    alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    allocs.push_back(p);
    bytes += (int64_t)b;
    return static_cast<T*>(p);
  }
  void release(void* p) {
    if (pool) ck(cudaFreeAsync(p, stream), "cudaFreeAsync");
    else ck(cudaFree(p), "cudaFree");
  }
  // create-time scratch: stream-ordered from the pool (freed without a host sync),
  // else cudaMalloc / synchronize + cudaFree
  void* tmp_get(size_t b) {
    void* p = nullptr;
    if (pool) ck(cudaMallocFromPoolAsync(&p, std::max<size_t>(b, 16), pool, stream), "cudaMallocFromPoolAsync");
    else ck(cudaMalloc(&p, std::max<size_t>(b, 16)), "cudaMalloc");
    return p;
  }
  void tmp_put(void* p) {
    if (!p) return;
    if (pool) {
      ck(cudaFreeAsync(p, stream), "cudaFreeAsync");
    } else {
      ck(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
      ck(cudaFree(p), "cudaFree");
    }
  }
  ~esnmf() {
    if (stream) cudaStreamSynchronize(stream);
    for (auto& g : gexec)
      if (g) cudaGraphExecDestroy(g);
    for (auto& r : prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (void* p : allocs) pool ? cudaFreeAsync(p, stream) : cudaFree(p);
    if (pool) {  // keep up to 24 GB mapped for the next handle, return the rest
      if (stream) cudaStreamSynchronize(stream);
      cudaMemPoolTrimTo(pool, (size_t)24 << 30);
    }
    if (aux) cudaStreamSynchronize(aux);
    for (cudaEvent_t e : {ev_ufork, ev_ujoin, ev_mfork, ev_mjoin, ev_vfork, ev_vjoin, ev_gfork, ev_gjoin,
                          ev_ugram})
      if (e) cudaEventDestroy(e);
    if (aux) cudaStreamDestroy(aux);
    if (maux) cudaStreamSynchronize(maux), cudaStreamDestroy(maux);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// enqueue on another stream for the lifetime of the object
struct OnStream {
  esnmf_t* h;
  cudaStream_t saved;
  OnStream(esnmf_t* h_, cudaStream_t s) : h(h_), saved(h_->stream) { h->stream = s; }
  ~OnStream() { h->stream = saved; }
};

// main -> side-stream dependency (the side stream waits for everything enqueued on main so far)
void fork_to(esnmf_t* h, cudaStream_t side, cudaEvent_t ev) {
  ck(cudaEventRecord(ev, h->stream), "cudaEventRecord(fork)");
  ck(cudaStreamWaitEvent(side, ev, 0), "cudaStreamWaitEvent(fork)");
}
// side stream -> main dependency
void join_from(esnmf_t* h, cudaStream_t side, cudaEvent_t ev) {
  ck(cudaEventRecord(ev, side), "cudaEventRecord(join)");
  ck(cudaStreamWaitEvent(h->stream, ev, 0), "cudaStreamWaitEvent(join)");
}
void fork_to_aux(esnmf_t* h, cudaEvent_t ev) { fork_to(h, h->aux, ev); }
void join_from_aux(esnmf_t* h, cudaEvent_t ev) { join_from(h, h->aux, ev); }
// the previous iteration's error/record kernels must finish before V is replaced
void join_metrics(esnmf_t* h) {
  if (!h->aux_pending) return;
  join_from(h, h->maux, h->ev_mjoin);
  h->aux_pending = false;
}

// ---------------------------------------------------------------- profiling
enum PhaseId { kVGram, kVSolve, kVFormZ, kVSpmm, kVSelect, kVRows, kUGram, kUSolve, kUFormZ, kUSpmm, kUSelect, kURows,
               kMetrics, kVHead, kVGather, kNumPhases };
const char* const kPhaseNames[kNumPhases] = {"V.gram",   "V.solve",  "V.form_z", "V.spmm",   "V.select",
                                             "V.rowview", "U.gram",  "U.solve",  "U.form_z", "U.spmm",
                                             "U.select", "U.rowview", "iter.metrics", "V.head", "V.gather"};

cudaEvent_t pool_event(esnmf_t* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  ck(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

// RAII event pair around one phase, recorded on the handle's stream
// Also an NVTX range named after the phase (host side: the launches of the phase,
// visible in Nsight Systems / Nsight Compute's NVTX filters; no cost without a tool)
struct Phase {
  esnmf_t* h;
  int id;
  cudaEvent_t a = nullptr;
  Phase(esnmf_t* h_, int id_) : h(h_), id(id_) {
    nvtxRangePushA(kPhaseNames[id]);
    if (h->prof_on) {
      a = pool_event(h);
      ck(cudaEventRecord(a, h->stream), "cudaEventRecord");
    }
  }
  ~Phase() {
    if (h->prof_on && a) {
      cudaEvent_t b = pool_event(h);
      cudaEventRecord(b, h->stream);
      h->prof.push_back({id, a, b});
    }
    nvtxRangePop();
  }
};

void prof_collect(esnmf_t* h) {
  for (auto& r : h->prof) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
    h->prof_ms[r.id] += ms;
    h->prof_calls[r.id] += 1;
    h->ev_pool.push_back(r.a);
    h->ev_pool.push_back(r.b);
  }
  h->prof.clear();
}

unsigned col_grid_x(int64_t maxcol) { return (unsigned)std::min<int64_t>(std::max<int64_t>(1, ceil_div(maxcol, 256)), 2048); }

void launch_scan_inplace(esnmf_t* h, int64_t* a, int64_t n, int64_t* total) {
  int64_t nb = ceil_div(n, kScanBlock);
  int64_t* bs = h->alloc<int64_t>(nb);  // create-time only
  ++h->nlaunch; k_blocksum_i64<<<(unsigned)nb, 256, 0, h->stream>>>(a, n, bs);
  ++h->nlaunch; k_scan_small<<<1, 1024, 0, h->stream>>>(bs, nb, total);
  ++h->nlaunch; k_scan_apply_i64<<<(unsigned)nb, 256, 0, h->stream>>>(a, n, bs);
  CKL("scan");
}

// ---------------------------------------------------------------- factors

void factor_alloc(esnmf_t* h, Factor& f, int64_t rows, int64_t cap, int kk = 0, int kp = 0) {
  if (!kk) kk = h->k, kp = h->kpad;
  f.rows = rows;
  f.cap = cap;
  f.cap_rows = std::min(rows, cap);
  f.colptr = h->alloc<int64_t>(kk + 1);
  f.row = h->alloc<int32_t>(cap);
  f.val = h->alloc<float>(cap);
  f.rowmap = h->alloc<int32_t>(rows);
  f.active = h->alloc<int32_t>(f.cap_rows);
  f.n_active = h->alloc<int64_t>(1);
  f.dense = h->alloc<float>(f.cap_rows * kp);
  CK(cudaMemsetAsync(f.colptr, 0, sizeof(int64_t) * (kk + 1), h->stream));
  CK(cudaMemsetAsync(f.rowmap, 0xFF, sizeof(int32_t) * rows, h->stream));
  CK(cudaMemsetAsync(f.n_active, 0, sizeof(int64_t), h->stream));
  CK(cudaMemsetAsync(f.dense, 0, sizeof(float) * f.cap_rows * kp, h->stream));
  f.has = false;
  f.maxcol = 0;
}

// undo the row view of the factor's current content (before it is replaced)
void factor_clear(esnmf_t* h, Factor& f, int kk = 0, int kp = 0) {
  if (!f.has) return;
  if (!kk) kk = h->k, kp = h->kpad;
  dim3 g(col_grid_x(f.maxcol), kk);
  ++h->nlaunch; k_clear_dense<<<g, 256, 0, h->stream>>>(f.colptr, f.row, f.rowmap, f.dense, kp);
  ++h->nlaunch; k_reset_rowmap<<<grid_for(f.cap_rows, 256, 4096), 256, 0, h->stream>>>(f.active, f.n_active, f.rowmap);
  CKL("factor_clear");
  f.has = false;
}

// build rowmap / active / dense from the column-major COO just written
void factor_build_rows(esnmf_t* h, Factor& f, int64_t maxcol, int kk = 0, int kp = 0) {
  if (!kk) kk = h->k, kp = h->kpad;
  f.maxcol = maxcol;
  dim3 g(col_grid_x(maxcol), kk);
  ++h->nlaunch; k_mark_rows<<<g, 256, 0, h->stream>>>(f.colptr, f.row, f.rowmap);
  const int64_t nb = ceil_div(f.rows, kRowBlock);
  int64_t* bc = reinterpret_cast<int64_t*>(h->red);  // scratch (nb <= red_cap)
  ++h->nlaunch; k_rows_count<<<(unsigned)nb, 256, 0, h->stream>>>(f.rowmap, f.rows, bc);
  ++h->nlaunch; k_scan_small<<<1, 1024, 0, h->stream>>>(bc, nb, f.n_active);
  ++h->nlaunch; k_rows_assign<<<(unsigned)nb, 256, 0, h->stream>>>(f.rowmap, f.rows, bc, f.active);
  ++h->nlaunch; k_scatter_dense<<<g, 256, 0, h->stream>>>(f.colptr, f.row, f.val, f.rowmap, f.dense, kp);
  CKL("factor_build_rows");
  f.has = true;
}

int64_t steady_maxcol(esnmf_t* h, int s, int64_t rows) {
  const int64_t t = h->tside[s];
  return t < 0 ? rows : std::min(rows, t);
}

// ---------------------------------------------------------------- kernels

void gram(esnmf_t* h, const Factor& f, double* G, int kk = 0, int kp = 0, double* partial = nullptr) {
  if (!kk) kk = h->k, kp = h->kpad, partial = h->gram_partial;
  const int k = kk;
  int64_t S = std::min<int64_t>(kMaxGramSeg, std::max<int64_t>(1, ceil_div(f.maxcol, 32)));
  int64_t seglen = std::max<int64_t>(1, ceil_div(f.maxcol, S));
  dim3 g(k, (unsigned)S);
  const int gb = (k + 31) / 32 * 32;  // <= 256
  ++h->nlaunch;
  if (f.maxcol * 4 >= f.rows && f.rows >= 256 && !getenv("ESNMF_GRAM_SPARSE")) {
    // long columns (dense U_0, unlimited t): straight from the dense active rows
    S = std::min<int64_t>(kMaxGramSegDense, std::max<int64_t>(1, ceil_div(f.rows, 512)));
    const unsigned nb = (unsigned)ceil_div(kp, 128);
    k_gram_dense<<<dim3((unsigned)S, nb, nb), 256, 0, h->stream>>>(f.dense, kp, k, f.n_active, partial);
  } else if (seglen >= 256) {  // long segments: thread groups split the entries
    const int ng = std::max(1, std::min(4, 512 / gb));
    k_gram_partial_groups<<<g, gb * ng, 0, h->stream>>>(f.colptr, f.row, f.val, f.rowmap, f.dense, kp, k, seglen,
                                                        partial, gb);
  } else {
    k_gram_partial<<<g, gb, 0, h->stream>>>(f.colptr, f.row, f.val, f.rowmap, f.dense, kp, k, seglen, partial);
  }
  ++h->nlaunch; k_gram_reduce<<<grid_for((int64_t)k * k, 256), 256, 0, h->stream>>>(partial, (int)S, k, G);
  CKL("gram");
}

template <int JB, bool PACKED>
void sweep_launch(esnmf_t* h, const double* G, double* eps, SweepCond sc) {
  const bool glob = h->k > 224;
  const size_t smem = sweep_smem_bytes(h->k, glob);
  auto kern = k_sweep_inverse<JB, PACKED>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ++h->nlaunch;
  kern<<<1, 1024, smem, h->stream>>>(G, h->k, h->rho, h->W, eps, h->flags, glob ? h->sweep_scratch : nullptr, sc);
  CKL("sweep_inverse");
}

void sweep(esnmf_t* h, const double* G, double* eps, SweepCond sc = SweepCond()) {
  const int JB = (h->k + 31) / 32;
  const bool packed = sweep_packed(h->k);
  static const bool scalar = getenv("ESNMF_SWEEP_SCALAR") != nullptr;
  if (JB >= 2 && h->k <= 256 && !scalar) {  // blocked sweep (k_solve.cuh)
    bool in_smem = false;
    const size_t smem = bsweep_smem_bytes(h->k, &in_smem);
    CK(cudaFuncSetAttribute(k_sweep_blocked, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    ++h->nlaunch;
    k_sweep_blocked<<<1, kBsThreads, smem, h->stream>>>(G, h->k, h->rho, h->W, eps, h->flags,
                                                         in_smem ? nullptr : h->sweep_scratch, sc);
    CKL("sweep_blocked");
    return;
  }
  if (JB <= 4) {  // register-resident matrix
    ++h->nlaunch;
    switch (JB) {
      case 1: k_sweep_regs<1><<<1, 1024, 0, h->stream>>>(G, h->k, h->rho, h->W, eps, h->flags, sc); break;
      case 2: k_sweep_regs<2><<<1, 1024, 0, h->stream>>>(G, h->k, h->rho, h->W, eps, h->flags, sc); break;
      case 3: k_sweep_regs<3><<<1, 1024, 0, h->stream>>>(G, h->k, h->rho, h->W, eps, h->flags, sc); break;
      default: k_sweep_regs<4><<<1, 1024, 0, h->stream>>>(G, h->k, h->rho, h->W, eps, h->flags, sc); break;
    }
    CKL("sweep_regs");
    return;
  }
  switch (JB) {
    case 5: packed ? sweep_launch<5, true>(h, G, eps, sc) : sweep_launch<5, false>(h, G, eps, sc); break;
    case 6: sweep_launch<6, true>(h, G, eps, sc); break;
    case 7: sweep_launch<7, true>(h, G, eps, sc); break;
    default: sweep_launch<8, true>(h, G, eps, sc); break;
  }
}

// sequential mode, after the block's product T H_2 W_22: subtract O_1 (H_1^T H_2) W_22
// (Eq. (7) / (8); k_seq.cuh).  V side: H = U, O = V; U side: H = V, O = U.
void seq_deflate(esnmf_t* h, int s) {
  const int b0 = h->seq_b * h->seq_k2;
  if (!h->ktot || b0 == 0) return;
  Side& sd = h->side[s];
  const Factor& H2 = s == ESNMF_SIDE_V ? h->U[h->ucur] : h->V;
  const Factor& H1 = s == ESNMF_SIDE_V ? h->FU : h->FV;
  const Factor& O1 = s == ESNMF_SIDE_V ? h->FV : h->FU;
  const int k2 = h->k;
  h->nlaunch += 3;
  k_seq_cross<<<dim3(b0, k2), 256, 0, h->stream>>>(H1.colptr, H1.row, H1.val, H2.rowmap, H2.dense, h->kpad, k2,
                                                   h->seqC);
  k_seq_m<<<grid_for((int64_t)b0 * k2, 256, 256), 256, 0, h->stream>>>(h->seqC, h->W, b0, k2, h->seqM);
  k_seq_deflate<<<grid_for(O1.cap_rows * k2, 256, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(
      O1.active, O1.n_active, O1.dense, h->kpf, b0, k2, h->seqM, sd.X, sd.ldx, sd.row0, sd.rows);
  CKL("seq_deflate");
}

void init_u0(esnmf_t* h, const float* user_u0, bool on_dev);

// block b is done (its seq_iters iterations, reading C12): append U_2, V_2 to
// U_1, V_1, refresh the record constants, restart from U_2 = U_0
void graph_reset(esnmf_t* h);

void seq_next_block(esnmf_t* h) {
  join_metrics(h);
  graph_reset(h);  // new block: b0, the frozen factors' bounds and U_0 change
  const int b0 = h->seq_b * h->seq_k2, k2 = h->k;
  const Factor& U2 = h->U[h->ucur];
  // record constants first (they need the old U_1, V_1): C_U, C_V into seqC / seqM
  if (b0 > 0) {
    h->nlaunch += 2;
    k_seq_cross<<<dim3(b0, k2), 256, 0, h->stream>>>(h->FU.colptr, h->FU.row, h->FU.val, U2.rowmap, U2.dense,
                                                     h->kpad, k2, h->seqC);
    k_seq_cross<<<dim3(b0, k2), 256, 0, h->stream>>>(h->FV.colptr, h->FV.row, h->FV.val, h->V.rowmap, h->V.dense,
                                                     h->kpad, k2, h->seqM);
  }
  // G_U2 = side V's G (the metrics' Gram of the final U_2), G_V2 = side U's G
  ++h->nlaunch;
  k_seq_consts<<<1, 256, 0, h->stream>>>(h->seqC, h->seqM, b0 * k2, h->scal + 2, h->side[ESNMF_SIDE_V].G,
                                         h->side[ESNMF_SIDE_U].G, k2, h->seqc);
  for (int q = 0; q < 2; ++q) {
    Factor& F = q == 0 ? h->FU : h->FV;
    const Factor& B = q == 0 ? U2 : h->V;
    factor_clear(h, F, h->ktot, h->kpf);
    h->nlaunch += 2;
    k_seq_append_entries<<<grid_for(B.cap, 256, (int64_t)h->num_sms * 8), 256, 0, h->stream>>>(
        B.colptr, B.row, B.val, k2, b0, F.colptr, F.row, F.val);
    k_seq_append_colptr<<<1, 256, 0, h->stream>>>(B.colptr, k2, b0, h->ktot, F.colptr);
    factor_build_rows(h, F, std::max(F.maxcol, B.maxcol), h->ktot, h->kpf);
  }
  CKL("seq_next_block");
  ++h->seq_b;
  h->seq_i = 0;
  factor_clear(h, h->U[0]);
  factor_clear(h, h->U[1]);
  init_u0(h, nullptr, false);  // U_2 = U_0 (k2 columns), ucur = 0
}

// V side: Z = U W written term-indexed (stride zs); the rows written by the
// previous call are zeroed first, and the active-term bitmap is rebuilt.
void form_z(esnmf_t* h, const Factor& f, const int* gate = nullptr) {
  const int zq = h->zs / 4;
  const int kpz = h->k == 1 ? 1 : h->kpad;  // zc row width
  if (h->zc) {  // narrow k: the compact z of the previous call is cleared with the same list
    ++h->nlaunch;
    k_zc_clear<<<grid_for(f.cap_rows * kpz, 256, (int64_t)h->num_sms * 8), 256, 0, h->stream>>>(h->zlist, h->zcount,
                                                                                               kpz, h->zc);
  }
  // gated launches (the Z-row gather as the paper-order tail's fallback) take
  // grid-stride grids of 4 blocks per SM: when the gate is off they cost a few
  // microseconds instead of thousands of blocks that exit at once
  const int64_t gcap = gate ? 4 : 32;
  ++h->nlaunch;
  k_zrows_clear<<<grid_for(f.cap_rows * zq, 256, (int64_t)h->num_sms * gcap), 256, 0, h->stream>>>(
      h->zlist, h->zcount, reinterpret_cast<float4*>(h->Z), zq, gate);
  const int CJ = (h->kpad + 31) / 32;
  unsigned grid = grid_for(f.cap_rows, 8, (int64_t)h->num_sms * (gate ? 4 : 64));
  if (h->ptail && !h->zc) {  // Z64 = U W is already there (form_z64): convert it
    ++h->nlaunch;
    k_form_z_from64<<<grid, 256, 0, h->stream>>>(f.n_active, f.active, h->k, h->zs, h->Z64, h->Z, h->zlist, h->zcount,
                                                 gate);
    CKL("form_z");
    return;
  }
#define ESNMF_FZ(cj)                                                                                          \
  case cj:                                                                                                    \
    ++h->nlaunch;                                                                                             \
    k_form_z<cj><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->zs, h->W, h->Z, \
                                              h->zlist, h->zcount, gate);                                     \
    break;
  switch (CJ) {
    ESNMF_FZ(1) ESNMF_FZ(2) ESNMF_FZ(3) ESNMF_FZ(4) ESNMF_FZ(5) ESNMF_FZ(6) ESNMF_FZ(7) ESNMF_FZ(8)
    default: fail(ESNMF_EINVAL, "k too large");
  }
#undef ESNMF_FZ
  if (h->zc) {
    ++h->nlaunch;
    k_zc_fill<<<grid_for(f.cap_rows * kpz, 256, (int64_t)h->num_sms * 8), 256, 0, h->stream>>>(
        h->zlist, h->zcount, h->Z, h->zs, kpz, h->zc);
  }
  if (h->ptail) {  // the gather reads only tail entries; U's row bitmap (urows_build) marks its active rows
    CKL("form_z");
    return;
  }
  CK(cudaMemsetAsync(h->tbits, 0, sizeof(uint32_t) * ceil_div(h->n, 32), h->stream));
  ++h->nlaunch;
  k_term_bits<<<grid_for(f.cap_rows, 256, 4096), 256, 0, h->stream>>>(f.active, f.n_active, h->tbits, gate);
  if (h->head_h > 0) {  // head terms go through the tensor cores (k_vhead.cuh), not the gather
    ++h->nlaunch;
    k_head_bits_clear<<<(unsigned)ceil_div(h->head_h, 256), 256, 0, h->stream>>>(h->headterm, h->head_h, h->tbits,
                                                                                  gate);
    if (!h->ptail) {  // (paper-order mode: k_vside_prep writes the Z chunks)
      ++h->nlaunch;
      k_zhead_prep<<<h->k, 256, 0, h->stream>>>(h->Z, h->zs, h->headterm, h->head_h, h->kn, h->amax_bits, h->zhead,
                                                h->colscale);
    }
  }
  CKL("form_z");
}

// (G lanes per Z row) x (CPL float4 per lane) = Z row stride / 4
void tail_layout(int kpad, int& G, int& CPL) {
  const int KQ = kpad / 4;
  if (KQ <= 4) { G = 4; CPL = 1; }
  else if (KQ <= 8) { G = 8; CPL = 1; }
  else if (KQ <= 16) { G = 8; CPL = 2; }
  else if (KQ <= 32) { G = 32; CPL = 1; }
  else { G = 32; CPL = 2; }
}

template <int G, int CPL, int U, int RG>
void tail_launch(esnmf_t* h, const int* gate) {
  Side& sd = h->side[ESNMF_SIDE_V];
  const float4* Z4 = reinterpret_cast<const float4*>(h->Z);
  const int64_t nwords = ceil_div(h->n, 32);
  const bool smem_bits = nwords * 4 <= 64 * 1024;
  const size_t smem = smem_bits ? nwords * 4 : 0;
  if (h->zs != 4 * G * CPL) fail(ESNMF_EINVAL, "Z row stride does not match the tail gather layout");
  // with a head: row-major staging (the head kernel adds its part and stores X);
  // without: column-major straight into X
  const bool trow = h->head_h > 0 || h->ptail;
  auto kern = trow ? k_spmm_tail<G, CPL, U, RG, true> : k_spmm_tail<G, CPL, U, RG, false>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t groups = ceil_div(sd.rows, RG);
  unsigned grid = (unsigned)std::min<int64_t>(ceil_div(groups, kTailThreads / 32), (int64_t)h->num_sms * kTailMinBlocks);
  ++h->nlaunch;
  kern<<<grid, kTailThreads, smem, h->stream>>>(sd.T.ptr, h->head_h > 0 ? h->nh : nullptr, sd.T.ent, sd.rows,
                                                h->ptail ? h->ubits : h->tbits, smem_bits ? (int)nwords : 0, Z4,
                                                h->zs / 4, h->kpad / 4,
                                                h->k, trow ? sd.Xt : sd.X, trow ? (int64_t)h->kpad : sd.ldx, gate);
  CKL("spmm_tail");
}

// U side: paper order, fp64 (A V) from the sparse V rows, then (A V) W
template <int CQ>
void spmm_terms_launch(esnmf_t* h) {
  Side& sd = h->side[ESNMF_SIDE_U];
  unsigned grid = (unsigned)std::min<int64_t>(ceil_div(sd.nitems, 8), (int64_t)h->num_sms * 8);
  auto* part = reinterpret_cast<unsigned long long*>(sd.partial);
  ++h->nlaunch;
  k_spmm_terms<CQ><<<grid, 256, 0, h->stream>>>(sd.items, sd.nitems, sd.item_slot, sd.T.ent, h->rsum, h->vbits,
                                                h->vmap, h->vent, h->vmax, h->W, h->k, h->kpad, sd.X, sd.ldx, part);
  if (sd.nsplit > 0) {
    ++h->nlaunch;
    k_terms_combine<CQ><<<grid_for(sd.nsplit, 8, 4096), 256, 0, h->stream>>>(sd.splits, sd.nsplit, part, h->rsum,
                                                                             h->vmax, h->W, h->k, h->kpad, sd.X,
                                                                             sd.ldx);
  }
  CKL("spmm_terms");
}

// fp32 copy of W and the conditioning flag choosing the fp32 or fp64 (Y W)
void uside_w_prep(esnmf_t* h) {
  h->nlaunch += 1;
  k_w_to_f32<<<grid_for((int64_t)h->k * h->kpad, 256, 256), 256, 0, h->stream>>>(h->W, h->k, h->kpad, h->W32);
  // fp32 / tensor-core (Y W) when kappa(G_V + eps I) <= u_kmax, else fp64 -- decided
  // on the device by the U side's sweep (SweepCond, flags[3])
  if (h->utc_kn) {
    ++h->nlaunch;
    k_utc_wprep<<<h->k, 128, 0, h->stream>>>(h->W, h->k, h->utc_kn, h->utc_kk, h->wtc, h->wtc_scale);
  }
  CKL("uside_w_prep");
}

// U side on one GPU: scatter from the active documents (k_uside_scatter.cuh)
template <int CQ>
void uside_scatter_launch(esnmf_t* h) {
  Side& su = h->side[ESNMF_SIDE_U];
  Side& sv = h->side[ESNMF_SIDE_V];
  Factor& V = h->V;
  ++h->nlaunch;
  if (h->head_h > 0 && !getenv("ESNMF_SCATTER_ROWS")) {  // by V's columns, head terms in shared memory
    const size_t smem = sizeof(unsigned long long) * h->head_h;
    CK(cudaFuncSetAttribute(k_uside_scatter_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int nd = kScatDocs;
    const dim3 g((unsigned)ceil_div(std::max<int64_t>(V.maxcol, 1), nd), h->k);
    k_uside_scatter_cols<<<g, 256, smem, h->stream>>>(V.colptr, V.row, V.val, sv.T.ptr, h->nh, sv.T.ent, h->headslot,
                                                      h->headterm, h->head_h, h->rsum_max, h->vmax, h->kpad, h->Yq,
                                                      nd);
  } else {
    k_uside_scatter<<<grid_for(V.cap_rows, 8, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(
        V.active, V.n_active, h->vmap, h->vent, sv.T.ptr, sv.T.ent, h->rsum_max, h->vmax, h->kpad, h->Yq);
  }
  // Gram + solve + W prep (uside_w_prep) ran on the aux stream beside the scatter
  join_from_aux(h, h->ev_ujoin);
  h->nlaunch += 2;
  // W32 staged in shared memory + per-warp transposed Y tiles (8 warps)
  const size_t smem = sizeof(float) * h->k * h->kpad + sizeof(float) * 8 * h->kpad * kFinRT;
  const int64_t rgroups = ceil_div(su.rows, kFinRT);
  if (h->utc_kn) {  // tensor cores (k_uside_tc.cuh)
    const size_t tsm = uside_tc_smem(h->utc_kn, h->utc_kk);
    CK(cudaFuncSetAttribute(k_uside_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    const int64_t ntiles = ceil_div(su.rows, kUtcM);
    const int acc = h->utc_kn <= 32 ? 32 : h->utc_kn <= 64 ? 64 : 128;
    k_uside_tc<<<(unsigned)std::min<int64_t>(ntiles, h->num_sms), kUtcThreads, tsm, h->stream>>>(
        su.rows, ntiles, h->rsum_max, h->vmax, h->wtc, h->wtc_scale, h->k, h->kpad, h->utc_kn, h->utc_kk, acc, h->Yq,
        su.X, su.ldx, h->flags + 3);
  } else if (h->kpad <= 128) {
    CK(cudaFuncSetAttribute(k_uside_finish_rt<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_uside_finish_rt<1><<<grid_for(rgroups, 8, (int64_t)h->num_sms * 3), 256, smem, h->stream>>>(
        su.rows, h->rsum_max, h->vmax, h->W32, h->k, h->kpad, h->Yq, su.X, su.ldx, h->flags + 3);
  } else if ((int)smem <= h->smem_optin) {
    CK(cudaFuncSetAttribute(k_uside_finish_rt<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_uside_finish_rt<2><<<grid_for(rgroups, 8, (int64_t)h->num_sms * 1), 256, smem, h->stream>>>(
        su.rows, h->rsum_max, h->vmax, h->W32, h->k, h->kpad, h->Yq, su.X, su.ldx, h->flags + 3);
  }
  // fp64 (Y W) for ill-conditioned systems -- and always when W does not fit in shared memory (k > ~224)
  const bool fits = (int)smem <= h->smem_optin;
  k_uside_finish<CQ><<<grid_for(su.rows, 8, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(
      su.rows, h->rsum_max, h->vmax, h->W, h->k, h->kpad, h->Yq, su.X, su.ldx, fits ? h->flags + 3 : nullptr);
  CKL("uside_scatter");
}

void spmm(esnmf_t* h, int s, const int32_t* rowmap, const int* gate = nullptr) {
  if (s == ESNMF_SIDE_V && h->zc) {  // narrow k: SpMM over A^T with the compact z (k_spmm_narrow)
    Side& sd = h->side[ESNMF_SIDE_V];
    const unsigned g = grid_for(sd.rows, 8, (int64_t)h->num_sms * 64);
    ++h->nlaunch;
    if (h->k == 1)
      k_spmm_narrow<1><<<g, 256, 0, h->stream>>>(sd.T.ptr, sd.T.ent, sd.rows, h->zc, h->k, sd.X, sd.ldx);
    else if (h->kpad == 4)
      k_spmm_narrow<4><<<g, 256, 0, h->stream>>>(sd.T.ptr, sd.T.ent, sd.rows, h->zc, h->k, sd.X, sd.ldx);
    else
      k_spmm_narrow<8><<<g, 256, 0, h->stream>>>(sd.T.ptr, sd.T.ent, sd.rows, h->zc, h->k, sd.X, sd.ldx);
    CKL("spmm_narrow");
    return;
  }
  if (s == ESNMF_SIDE_U && !h->sharded) {
    switch ((h->k + 31) / 32) {
      case 1: uside_scatter_launch<1>(h); break;
      case 2: uside_scatter_launch<2>(h); break;
      case 3: uside_scatter_launch<3>(h); break;
      case 4: uside_scatter_launch<4>(h); break;
      case 5: uside_scatter_launch<5>(h); break;
      case 6: uside_scatter_launch<6>(h); break;
      case 7: uside_scatter_launch<7>(h); break;
      default: uside_scatter_launch<8>(h); break;
    }
    return;
  }
  if (s == ESNMF_SIDE_U) {
    switch ((h->k + 31) / 32) {
      case 1: spmm_terms_launch<1>(h); break;
      case 2: spmm_terms_launch<2>(h); break;
      case 3: spmm_terms_launch<3>(h); break;
      case 4: spmm_terms_launch<4>(h); break;
      case 5: spmm_terms_launch<5>(h); break;
      case 6: spmm_terms_launch<6>(h); break;
      case 7: spmm_terms_launch<7>(h); break;
      default: spmm_terms_launch<8>(h); break;
    }
    return;
  }
  const int KQ = h->kpad / 4;
  // layouts must match tail_layout() (the Z row stride)
  if (KQ <= 4) tail_launch<4, 1, 2, 4>(h, gate);
  else if (KQ <= 8) tail_launch<8, 1, 2, 4>(h, gate);
  else if (KQ <= 16) tail_launch<8, 2, 2, 2>(h, gate);
  else if (KQ <= 32) tail_launch<32, 1, 4, 4>(h, gate);
  else tail_launch<32, 2, 4, 2>(h, gate);
}

// ---- V row-CSR for the U side (k_spmm_terms.cuh) ----
// the single-GPU U side with a head scatters by V's columns (k_uside_scatter_cols):
// V's row-CSR is only needed by the row-driven scatter and the sharded term kernel.
// Without it the scatter waits on an event after the U side's Gram (on aux) instead:
// launched beside the scatter's full grid, the one-CTA solve found no SM until the
// scatter drained (2.12 -> 2.17 ms at Large when the row-CSR build was simply
// skipped); released together, the solve's higher-priority CTA is placed first.
// ESNMF_VROWS=1 builds the row-CSR anyway (the old ~0.04 ms gap, for measurement).
bool need_vrows(esnmf_t* h) {
  static const bool force = getenv("ESNMF_VROWS") != nullptr;
  return h->sharded || h->head_h == 0 || getenv("ESNMF_SCATTER_ROWS") || force;
}

void vrows_clear(esnmf_t* h) {
  Factor& f = h->V;
  if (!f.has || !need_vrows(h)) return;
  ++h->nlaunch;
  k_vrows_clear<<<grid_for(f.cap_rows, 256, 4096), 256, 0, h->stream>>>(f.active, f.n_active, h->vmap, h->vbits);
  CKL("vrows_clear");
}

void vrows_build(esnmf_t* h) {
  Factor& f = h->V;
  if (!need_vrows(h)) {
    CK(cudaMemsetAsync(h->vmax, 0, sizeof(uint32_t), h->stream));
    ++h->nlaunch;
    k_vmax_only<<<grid_for(f.cap, 256, (int64_t)h->num_sms * 2), 256, 0, h->stream>>>(f.colptr, f.val, h->k, h->vmax);
    CKL("vmax_only");
    return;
  }
  const int64_t nr = f.cap_rows + 1;
  CK(cudaMemsetAsync(h->vrptr, 0, sizeof(int64_t) * nr, h->stream));
  dim3 g(col_grid_x(f.maxcol), h->k);
  ++h->nlaunch;
  k_vrows_count<<<g, 256, 0, h->stream>>>(f.colptr, f.row, f.rowmap, h->vrptr);
  const int64_t nb = ceil_div(nr, kScanBlock);
  h->nlaunch += 3;
  k_blocksum_i64<<<(unsigned)nb, 256, 0, h->stream>>>(h->vrptr, nr, h->vscan);
  k_scan_small<<<1, 1024, 0, h->stream>>>(h->vscan, nb, h->vscan + nb);
  k_scan_apply_i64<<<(unsigned)nb, 256, 0, h->stream>>>(h->vrptr, nr, h->vscan);
  CK(cudaMemcpyAsync(h->vcur, h->vrptr, sizeof(int64_t) * nr, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaMemsetAsync(h->vmax, 0, sizeof(uint32_t), h->stream));
  h->nlaunch += 2;
  k_vrows_scatter<<<g, 256, 0, h->stream>>>(f.colptr, f.row, f.val, f.rowmap, h->vcur, h->vent, h->vmax);
  k_vrows_finish<<<grid_for(f.cap_rows, 256, 4096), 256, 0, h->stream>>>(f.active, f.n_active, h->vrptr, h->vent,
                                                                         h->vmap, h->vbits);
  CKL("vrows_build");
}

// clamp + per-column top-t of side s's LS into factor `out` (column-major COO)
// the selection over a column-major buffer X (ldx x kc, `rows` rows used) into
// (colptr_out[kc+1], row_out, val_out); per-column top-t, or with kc = 1 over a
// flat view of the whole factor
void select_core(esnmf_t* h, Side& sd, const float* X, int64_t ldx, int64_t rows, int kc, int64_t row0, int64_t t,
                 bool use_pred, int64_t* colptr_out, int32_t* row_out, float* val_out, int64_t* peak_out) {
  const int k = kc;
  if (rows == 0) fail(ESNMF_EINVAL, "empty shard");
  const int64_t nch = std::max<int64_t>(1, ceil_div(rows, kSelChunk));
  const int64_t nseg = nch * kSelSegs;  // per-(column, segment) output counts
  CK(cudaMemsetAsync(sd.hist, 0, sizeof(uint32_t) * k * kNumBins, h->stream));
  CK(cudaMemsetAsync(sd.cand_fill, 0, sizeof(int32_t) * k, h->stream));
  dim3 g((unsigned)nch, k);
  // two-pass path: the [k][t] list must fit and the kept set of a column must fit k_sel_final's smem
  // (not for the flat whole-factor view, rows > ldx: its one column would run k_sel_final in one block)
  const bool fast = sd.above && t >= 0 && t <= kSelFastT && t * kc <= sd.above_t * h->k && rows <= sd.ldx;
  if (fast && sd.pred && use_pred) {
    // one pass over X in steady state: histogram + candidates above the predicted
    // threshold (k_sel_pred_final); columns whose prediction failed take the
    // second pass (k_sel_collect2 + k_sel_final)
    CK(cudaMemsetAsync(sd.pfill, 0, sizeof(int32_t) * k, h->stream));
    ++h->nlaunch;
    k_sel_hist<<<g, 256, 0, h->stream>>>(X, ldx, rows, sd.hist, sd.pred, row0, sd.pcand, sd.pfill,
                                         sd.pcap);
    ++h->nlaunch; k_sel_threshold<<<k, 1024, 0, h->stream>>>(sd.hist, t, sd.sel);
    ++h->nlaunch;
    k_sel_colptr_kept<<<1, 256, 0, h->stream>>>(sd.sel, k, t, colptr_out, peak_out);
    int32_t* done = sd.pfill + k;
    const size_t psm = sizeof(uint64_t) * (kSelFastT + kSelCap);
    CK(cudaFuncSetAttribute(k_sel_pred_final, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
    ++h->nlaunch;
    k_sel_pred_final<<<k, 1024, psm, h->stream>>>(sd.sel, std::max<int64_t>(t, 1), sd.pcand, sd.pfill, sd.pcap,
                                                  colptr_out, row_out, val_out, done, sd.pred);
    CK(cudaMemsetAsync(sd.above_fill, 0, sizeof(int32_t) * 2 * k, h->stream));
    int32_t* bfill = sd.above_fill + k;
    ++h->nlaunch;
    // (second pass for the columns whose prediction failed: 16 blocks per column
    // loop over the chunks, cheap when every column is done)
    const dim3 gf((unsigned)std::min<int64_t>(nch, 16), k);
    k_sel_collect2<<<gf, 256, 0, h->stream>>>(X, ldx, rows, row0, sd.sel, std::max<int64_t>(t, 1),
                                              sd.above, sd.above_fill, sd.bucket, bfill, done);
    CK(cudaFuncSetAttribute(k_sel_final, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelFinalSmem));
    ++h->nlaunch;
    k_sel_final<<<k, 1024, kSelFinalSmem, h->stream>>>(X, ldx, rows, row0, sd.sel,
                                                       std::max<int64_t>(t, 1), sd.above, sd.above_fill,
                                                       sd.bucket, bfill, colptr_out, row_out, val_out, done,
                                                       sd.pred);
    CKL("select2");
    return;
  }
  ++h->nlaunch; k_sel_hist<<<g, 256, 0, h->stream>>>(X, ldx, rows, sd.hist);
  ++h->nlaunch; k_sel_threshold<<<k, 1024, 0, h->stream>>>(sd.hist, t, sd.sel);
  if (fast) {  // two passes over X (k_sel_collect2 + k_sel_final)
    ++h->nlaunch;
    k_sel_colptr_kept<<<1, 256, 0, h->stream>>>(sd.sel, k, t, colptr_out, peak_out);
    CK(cudaMemsetAsync(sd.above_fill, 0, sizeof(int32_t) * 2 * k, h->stream));
    int32_t* bfill = sd.above_fill + k;
    ++h->nlaunch;
    k_sel_collect2<<<g, 256, 0, h->stream>>>(X, ldx, rows, row0, sd.sel, std::max<int64_t>(t, 1),
                                             sd.above, sd.above_fill, sd.bucket, bfill);
    CK(cudaFuncSetAttribute(k_sel_final, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelFinalSmem));
    ++h->nlaunch;
    k_sel_final<<<k, 1024, kSelFinalSmem, h->stream>>>(X, ldx, rows, row0, sd.sel,
                                                       std::max<int64_t>(t, 1), sd.above, sd.above_fill,
                                                       sd.bucket, bfill, colptr_out, row_out, val_out);
    CKL("select2");
    return;
  }
  // candidate list per column: kSelCap keys (sorted on chip); a flat whole-factor
  // view (one column) gets the whole buffer, so its bucket usually fits and the
  // radix levels run over the list instead of over X
  const int ccap = kc == 1 ? (int)std::min<int64_t>((int64_t)h->k * sd.ccap, INT32_MAX) : sd.ccap;
  if (peak_out) { ++h->nlaunch; k_sel_npos_sum<<<1, 256, 0, h->stream>>>(sd.sel, k, peak_out); }
  ++h->nlaunch; k_sel_collect<<<g, 256, 0, h->stream>>>(X, ldx, rows, row0, sd.sel, sd.cand, sd.cand_fill,
                                          sd.chunk_cnt, nseg, ccap);
  ++h->nlaunch; k_sel_refine<<<k, 1024, 0, h->stream>>>(X, ldx, rows, row0, sd.sel, sd.cand, sd.cand_fill,
                                          sd.chunk_cnt, nseg, sd.kthr, ccap);
  {  // columns whose threshold bucket overflowed kSelCap: exact radix levels
    CK(cudaMemsetAsync(sd.hist, 0, sizeof(uint32_t) * k * kNumBins, h->stream));
    ++h->nlaunch; k_sel_lvl_init<<<1, 256, 0, h->stream>>>(sd.sel, sd.cand_fill, k, sd.lvl, ccap);
    const int shifts[5] = {39, 32, 20, 8, 0}, widths[5] = {12, 7, 12, 12, 8};
    const dim3 gc((unsigned)ceil_div(ccap, 2048), k);
    for (int lv = 0; lv < 5; ++lv) {
      h->nlaunch += 3;
      k_sel_lvl_hist<<<g, 256, 0, h->stream>>>(X, ldx, rows, row0, sd.sel, sd.lvl, shifts[lv], widths[lv], sd.hist);
      k_sel_lvl_hist_cand<<<gc, 256, 0, h->stream>>>(sd.cand, sd.cand_fill, ccap, sd.lvl, shifts[lv], widths[lv],
                                                     sd.hist);
      k_sel_lvl_pick<<<k, 256, 0, h->stream>>>(sd.hist, shifts[lv], widths[lv], lv == 4, sd.lvl);
    }
    ++h->nlaunch;
    k_sel_cand_count<<<gc, 256, 0, h->stream>>>(sd.cand, sd.cand_fill, ccap, sd.lvl, row0, sd.chunk_cnt, nseg,
                                               sd.kthr);
    ++h->nlaunch; k_sel_lvl_count<<<g, 256, 0, h->stream>>>(X, ldx, rows, row0, sd.sel, sd.lvl, sd.chunk_cnt, nseg,
                                                            sd.kthr);
  }
  if (kc == 1 && nseg > 8 * kScanBlock) {  // one long (flat whole-factor) column: multi-block scan
    const int64_t nb = ceil_div(nseg, kScanBlock);
    if (nb > kSelScanMax) fail(ESNMF_EINVAL, "selection: flat view too long");
    h->nlaunch += 3;
    k_blocksum_i64<<<(unsigned)nb, 256, 0, h->stream>>>(sd.chunk_cnt, nseg, sd.scanbuf);
    k_scan_small<<<1, 1024, 0, h->stream>>>(sd.scanbuf, nb, sd.coltot);
    k_scan_apply_i64<<<(unsigned)nb, 256, 0, h->stream>>>(sd.chunk_cnt, nseg, sd.scanbuf);
  } else {
    ++h->nlaunch; k_sel_scan_cols<<<k, 1024, 0, h->stream>>>(sd.chunk_cnt, nseg, sd.coltot);
  }
  ++h->nlaunch; k_sel_colptr<<<1, 256, 0, h->stream>>>(sd.coltot, k, colptr_out);
  ++h->nlaunch; k_sel_write<<<g, 256, 0, h->stream>>>(X, ldx, rows, row0, sd.sel, sd.kthr, colptr_out,
                                        sd.chunk_cnt, nseg, row_out, val_out);
  CKL("select");
}

// flat selection indices (c * ldx + row, ascending) -> per-column colptr (one
// binary search per column) ...
__global__ void k_whole_colptr(const int32_t* __restrict__ idx, const int64_t* __restrict__ flat_colptr,
                               int64_t ldx, int k, int64_t* __restrict__ colptr) {
  const int64_t nnz = flat_colptr[1];
  for (int c = threadIdx.x; c <= k; c += blockDim.x) {
    int64_t lo = 0, hi = nnz;
    const int64_t key = (int64_t)c * ldx;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)(uint32_t)idx[mid] < key) lo = mid + 1; else hi = mid;
    }
    colptr[c] = lo;
  }
}

// ... and rows in place (after k_whole_colptr has read the flat indices)
__global__ void k_whole_rows(int32_t* __restrict__ idx, const int64_t* __restrict__ flat_colptr, int64_t ldx) {
  const int64_t nnz = flat_colptr[1];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x)
    idx[q] = (int32_t)((uint32_t)idx[q] % (uint32_t)ldx);  // k * ldx < 2^31: 32-bit division
}

void vhead_launch(esnmf_t* h, bool rerun);

// V side after a fused head epilogue: select from the candidates, histogram
// path only for the columns whose prediction failed
void select_fused(esnmf_t* h, Side& sd, Factor& out) {
  const int64_t t = h->tside[ESNMF_SIDE_V];
  const int k = h->k;
  int32_t* done = sd.pfill + k;
  h->nlaunch += 2;
  k_sel_npos_colptr<<<1, 256, 0, h->stream>>>(sd.npos, k, t, out.colptr, sd.peak);
  CK(cudaFuncSetAttribute(k_sel_pred_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPredSortSmem));
  k_sel_pred_sort<<<k, 1024, kPredSortSmem, h->stream>>>(sd.npos, t, sd.pcand, sd.pfill, sd.pcap, out.colptr, out.row,
                                                         out.val, done, sd.pred);
  if (sd.xdeferred) {  // the head wrote no X: write it now if a column needs its exact path
    sd.xdeferred = false;
    ++h->nlaunch;
    k_any_undone<<<1, 256, 0, h->stream>>>(done, k, sd.xneed);
    vhead_launch(h, true);
  }
  // failed columns: histogram, threshold, collect, final (done columns return at
  // once; 16 blocks per column loop over the chunks, so the usual all-done case costs
  // a few microseconds per launch instead of a full grid of empty blocks)
  const int64_t nch = std::max<int64_t>(1, ceil_div(sd.rows, kSelChunk));
  dim3 g((unsigned)std::min<int64_t>(nch, 16), k);
  CK(cudaMemsetAsync(sd.hist, 0, sizeof(uint32_t) * k * kNumBins, h->stream));
  CK(cudaMemsetAsync(sd.above_fill, 0, sizeof(int32_t) * 2 * k, h->stream));
  int32_t* bfill = sd.above_fill + k;
  h->nlaunch += 4;
  k_sel_hist<<<g, 256, 0, h->stream>>>(sd.X, sd.ldx, sd.rows, sd.hist, nullptr, 0, nullptr, nullptr, 0, done);
  k_sel_threshold<<<k, 1024, 0, h->stream>>>(sd.hist, t, sd.sel);
  k_sel_collect2<<<g, 256, 0, h->stream>>>(sd.X, sd.ldx, sd.rows, sd.row0, sd.sel, std::max<int64_t>(t, 1), sd.above,
                                           sd.above_fill, sd.bucket, bfill, done);
  CK(cudaFuncSetAttribute(k_sel_final, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelFinalSmem));
  k_sel_final<<<k, 1024, kSelFinalSmem, h->stream>>>(sd.X, sd.ldx, sd.rows, sd.row0, sd.sel, std::max<int64_t>(t, 1),
                                                     sd.above, sd.above_fill, sd.bucket, bfill, out.colptr, out.row,
                                                     out.val, done, sd.pred);
  CKL("select_fused");
}

// clamp + top-t of side s's LS into factor `out` (column-major COO)
void select_topt(esnmf_t* h, int s, Factor& out) {
  Side& sd = h->side[s];
  const int64_t t = h->tside[s];
  if (sd.fused) {
    sd.fused = false;
    select_fused(h, sd, out);
    return;
  }
  if (!h->whole) {
    select_core(h, sd, sd.X, sd.ldx, sd.rows, h->k, sd.row0, t, true, out.colptr, out.row, out.val, sd.peak);
    return;
  }
  // Alg. 2 as printed: one selection over the flat k x ldx buffer (padding rows are 0)
  select_core(h, sd, sd.X, (int64_t)h->k * sd.ldx, (int64_t)h->k * sd.ldx, 1, 0, t, false, h->wcolptr, out.row,
              out.val, sd.peak);
  h->nlaunch += 2;
  k_whole_colptr<<<1, 256, 0, h->stream>>>(out.row, h->wcolptr, sd.ldx, h->k, out.colptr);
  k_whole_rows<<<grid_for(out.cap, 256, (int64_t)h->num_sms * 8), 256, 0, h->stream>>>(out.row, h->wcolptr, sd.ldx);
  CKL("whole_split");
}

void select_merge(esnmf_t* h, int s, Factor& out);

// V side, head terms on the tensor cores: X += A^T[:, head] Z[head, :]
int head_stage_bytes_host(int kn) {
  return (int)((kHeadABytes + (uint32_t)kn * kHeadK * 4 + kHeadRawBytes + 1023u) & ~1023u);
}
int head_stages(int kn) { return std::max(2, std::min(6, (220 * 1024) / head_stage_bytes_host(kn))); }

// rerun: the gated second launch of select_fused (no fused pass, X written, all
// CTAs return at once unless sv.xneed is set)
template <int ST>
void vhead_launch_st(esnmf_t* h, bool rerun) {
  Side& sv = h->side[ESNMF_SIDE_V];
  const int smem = ST * head_stage_bytes_host(h->kn) + 1024;
  const unsigned grid = (unsigned)std::min<int64_t>(h->head_ntiles, h->num_sms);
  ++h->nlaunch;
  if (rerun) {
    auto kern = k_vhead_otf<ST, false>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kHeadOtfThreads, smem, h->stream>>>(h->atile, h->head_nd, h->hoff, h->hseg, h->amax_bits, h->zhead,
                                                     h->colscale, sv.rows, h->head_ntiles, h->head_nchunks, h->k,
                                                     h->kn, h->head_acc_cols, sv.X, sv.ldx, sv.Xt, h->kpad, SelFuse{},
                                                     h->ytile, h->wbuf, h->ptail ? h->nyc : 0,
                                                     h->ptail ? h->flags + 4 : nullptr, 1, sv.xneed);
    CKL("vhead_rerun");
    return;
  }
  // selection pass 1 in the epilogue (k_sel_pred_sort) when the V side takes the
  // predicted-threshold path: per-column top-t, t <= kSelFastT, one GPU.  Round 1
  // measured it slower (+0.14 ms on the head for ~0.1 ms saved); since the head's
  // epilogue waits on the (Y_tail W) chunks too it fits: head +0.03 ms, select
  // -0.10 ms at Large (2.19 -> 2.12 ms).  ESNMF_FUSED_SELECT=0 turns it off.
  const int64_t t = h->tside[ESNMF_SIDE_V];
  const char* fs_env = getenv("ESNMF_FUSED_SELECT");
  sv.fused = sv.pred && !h->whole && !h->sharded && t >= 0 && t <= kSelFastT && t <= sv.above_t &&
             !(h->ktot && h->seq_b > 0) &&  // Alg. 3 deflates X after this kernel
             h->kn <= 128 &&                 // <= 4 column chunks per epilogue warp
             ceil_div(h->head_ntiles, std::min<int64_t>(h->head_ntiles, h->num_sms)) < 65536 &&  // 16-bit counts
             !(fs_env && atoi(fs_env) == 0);
  SelFuse fz{};
  if (sv.fused) {
    CK(cudaMemsetAsync(sv.pfill, 0, sizeof(int32_t) * h->k, h->stream));
    CK(cudaMemsetAsync(sv.npos, 0, sizeof(int32_t) * h->k, h->stream));
    fz = SelFuse{sv.pred, sv.npos, sv.pcand, sv.pfill, sv.pcap, sv.row0};
  }
  // the LS buffer is written later, and only if needed (esnmf_options.keep_ls)
  sv.xdeferred = sv.fused && !h->keep_ls && !h->force_ls;
  sv.ls_stored = !sv.xdeferred;
  auto kern = sv.fused ? k_vhead_otf<ST, true> : k_vhead_otf<ST, false>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kHeadOtfThreads, smem, h->stream>>>(h->atile, h->head_nd, h->hoff, h->hseg, h->amax_bits, h->zhead,
                                                   h->colscale,
                                                   sv.rows, h->head_ntiles, h->head_nchunks, h->k, h->kn,
                                                   h->head_acc_cols, sv.X, sv.ldx, sv.Xt, h->kpad,
                                                   fz, h->ytile, h->wbuf, h->ptail ? h->nyc : 0,
                                                   h->ptail ? h->flags + 4 : nullptr, sv.xdeferred ? 0 : 1, nullptr);
  CKL("vhead");
}

void vhead_launch(esnmf_t* h, bool rerun) {
  switch (head_stages(h->kn)) {
    case 2: vhead_launch_st<2>(h, rerun); break;
    case 3: vhead_launch_st<3>(h, rerun); break;
    case 4: vhead_launch_st<4>(h, rerun); break;
    case 5: vhead_launch_st<5>(h, rerun); break;
    default: vhead_launch_st<6>(h, rerun); break;
  }
}

// Choose the head (create time): the terms of largest document frequency
// (row lengths of A, global), at least `min_df` of the documents each, a
// multiple of 64 terms, at most kHeadMax; or `want` terms when want > 0.
// kpad <= 8 on one GPU: the V side runs k_spmm_narrow (no head, no padded Z gather)
bool narrow_v(esnmf_t* h) { return h->kpad <= 8 && !h->sharded && !getenv("ESNMF_NO_NARROW"); }

void head_setup(esnmf_t* h, const std::vector<int64_t>& hptr, int32_t want) {
  if (narrow_v(h)) return;  // narrow k: the V side is an SpMM with a compact z (k_spmm_narrow)
  // the paper-order tail needs the term id in 24 bits of a packed entry
  h->ptail = h->n < (1LL << kVtTermBits) && !getenv("ESNMF_ZTAIL");
  const char* env = getenv("ESNMF_HEAD");
  if (env && env[0]) want = atoi(env);
  if (want == 0 && !h->ptail) return;
  const int64_t n = h->n;
  // terms by document frequency, descending, ties to the lower term id; only the
  // first hh (<= kHeadMax) are ever used, so only those are put in order
  auto df_of = [&](int32_t t) { return hptr[t + 1] - hptr[t]; };
  auto by_df = [&](int32_t a, int32_t b) {
    const int64_t da = df_of(a), db = df_of(b);
    return da != db ? da > db : a < b;
  };
  std::vector<int32_t> order;
  int64_t hh;
  if (want >= 0) {
    hh = std::min<int64_t>(want, n);
    order.resize(n);
    for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)i;
    const int64_t top = std::min<int64_t>(hh, kHeadMax);
    std::partial_sort(order.begin(), order.begin() + top, order.end(), by_df);
  } else {
    // document-frequency threshold of a head term.  Z-gather tail: 1.5 % (the
    // dense-tile cost balanced a 400-byte gather per active entry).  Paper-order
    // tail: a tail entry costs nnz(U row) products instead, so the head keeps only
    // the densest term bands
    double frac = 0.015;
    const char* fe = getenv("ESNMF_HEAD_DF");
    if (fe && fe[0]) frac = atof(fe);
    const double min_df = std::max(1.0, frac * (double)h->m);
    for (int64_t i = 0; i < n; ++i)
      if ((double)df_of((int32_t)i) >= min_df) order.push_back((int32_t)i);
    std::sort(order.begin(), order.end(), by_df);
    hh = (int64_t)order.size();
  }
  hh = std::min<int64_t>(hh, kHeadMax) / kHeadK * kHeadK;
  if (hh < kHeadK && !h->ptail) return;
  Side& sv = h->side[ESNMF_SIDE_V];
  h->kn = (h->k + 15) / 16 * 16;
  {  // TMEM columns per accumulator (two): kn, or 2 kn when wide (head_wide)
    const int cols = head_wide(h->kn) ? 2 * h->kn : h->kn;
    h->head_acc_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : 256;
  }
  h->head_h = (int)hh;
  h->head_nchunks = (int)(hh / kHeadK);
  h->head_ntiles = ceil_div(std::max<int64_t>(sv.rows, 1), kHeadM);
  std::vector<int32_t> slot(n, -1);
  for (int64_t s = 0; s < hh; ++s) slot[order[s]] = (int32_t)s;
  h->headterm = h->alloc<int32_t>(std::max<int64_t>(hh, 1));
  h->headslot = h->alloc<int32_t>(n);
  if (hh > 0) CK(cudaMemcpyAsync(h->headterm, order.data(), sizeof(int32_t) * hh, cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(h->headslot, slot.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, h->stream));
  h->zhead = h->alloc<uint8_t>(std::max<int64_t>(1, (int64_t)h->head_nchunks * h->kn * kHeadK * 4));
  sv.Xt = h->alloc<float>(std::max<int64_t>(sv.rows, 1) * h->kpad);  // (paper-order mode: the fallback's)
  sv.xneed = h->alloc<int>(1);
  h->colscale = h->alloc<float>(h->kn);
  h->amax_bits = h->alloc<unsigned>(1);
  CK(cudaMemsetAsync(h->zhead, 0, std::max<size_t>(1, (size_t)h->head_nchunks * h->kn * kHeadK * 4), h->stream));
  CK(cudaMemsetAsync(h->colscale, 0, sizeof(float) * h->kn, h->stream));
  CK(cudaMemsetAsync(h->amax_bits, 0, sizeof(unsigned), h->stream));
  // rows of A^T: head entries first (stable), so the tail reads skip them
  h->nh = h->alloc<int32_t>(std::max<int64_t>(sv.rows, 1));
  if (sv.T.nnz > 0 && hh > 0) {
    int2* tmp = static_cast<int2*>(h->tmp_get(sizeof(int2) * sv.T.nnz));
    ++h->nlaunch;
    k_reorder_head<<<grid_for(sv.rows, 8, (int64_t)h->num_sms * 32), 256, 0, h->stream>>>(
        sv.T.ptr, sv.T.ent, sv.rows, h->headslot, tmp, h->nh);
    CK(cudaMemcpyAsync(sv.T.ent, tmp, sizeof(int2) * sv.T.nnz, cudaMemcpyDeviceToDevice, h->stream));
    h->tmp_put(tmp);
  } else {
    CK(cudaMemsetAsync(h->nh, 0, sizeof(int32_t) * std::max<int64_t>(sv.rows, 1), h->stream));
  }
  ++h->nlaunch;
  k_absmax_ent<<<grid_for(std::max<int64_t>(sv.T.nnz, 1), 256, (int64_t)h->num_sms * 8), 256, 0, h->stream>>>(
      sv.T.ent, sv.T.nnz, h->amax_bits);
  if (h->ptail) {
    h->rowsum_bits = h->alloc<unsigned>(1);
    CK(cudaMemsetAsync(h->rowsum_bits, 0, sizeof(unsigned), h->stream));
    ++h->nlaunch;
    k_doc_rowsum_max<<<grid_for(std::max<int64_t>(sv.rows, 1), 8, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(
        sv.T.ptr, sv.T.ent, sv.rows, h->rowsum_bits);
  }
  if (h->sharded) {
    // the scales derived from max|A| and the largest document row sum must be the
    // same on every rank (every rank then rounds exactly as one GPU would)
    h->gmax_buf = h->alloc<uint32_t>(4 * (h->world + 1));
    CK(cudaMemsetAsync(h->gmax_buf, 0, sizeof(uint32_t) * 4 * (h->world + 1), h->stream));
    CK(cudaMemcpyAsync(h->gmax_buf, h->amax_bits, 4, cudaMemcpyDeviceToDevice, h->stream));
    if (h->rowsum_bits) CK(cudaMemcpyAsync(h->gmax_buf + 1, h->rowsum_bits, 4, cudaMemcpyDeviceToDevice, h->stream));
    if (h->comm.allgather(h->comm.ctx, h->gmax_buf, h->gmax_buf + 4, 16, h->stream) != 0)
      fail(ESNMF_ECOMM, "allgather(scales) failed");
    unsigned* rs = h->rowsum_bits ? h->rowsum_bits : h->gmax_buf + 2;
    ++h->nlaunch;
    k_rank_max2<<<1, 1, 0, h->stream>>>(h->gmax_buf + 4, h->world, h->amax_bits, rs);
  }
  // the densest chunks as dense tiles (bulk-copied as they are) ...
  if (hh > 0) {
    // 8 dense chunks measured best at Large (0.62 ms vs 0.64 for 4, 0.77 for all 16);
    // capped at 4 GB of dense tiles
    int nd = (int)std::min<int64_t>(512 / kHeadK, (int64_t)(4LL << 30) / std::max<int64_t>(1, h->head_ntiles * kHeadABytes));
    const char* de = getenv("ESNMF_HEAD_DENSE");
    if (de && de[0]) nd = atoi(de);
    h->head_nd = std::max(0, std::min(nd, h->head_nchunks));
    if (h->head_nd > 0) {
      const size_t ab = (size_t)h->head_ntiles * h->head_nd * kHeadABytes;
      h->atile = h->alloc<uint8_t>((int64_t)ab);
      const int smem = kHeadDenseG * (int)kHeadABytes;
      CK(cudaFuncSetAttribute(k_head_dense_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      ++h->nlaunch;
      k_head_dense_tiles<<<dim3((unsigned)h->head_ntiles, (unsigned)ceil_div(h->head_nd, kHeadDenseG)), 512, smem,
                           h->stream>>>(sv.T.ptr, h->nh, sv.T.ent, sv.rows, h->headslot, h->amax_bits, h->head_nd,
                                        h->atile);
    }
  }
  // ... and the others as a tiled copy of their entries: one run per (tile, chunk)
  {
    const int nsp = h->head_nchunks - h->head_nd;
    const int64_t nseg = h->head_ntiles * nsp;
    h->hoff = h->alloc<int64_t>(nseg + 1);
    CK(cudaMemsetAsync(h->hoff, 0, sizeof(int64_t) * (nseg + 1), h->stream));
    if (nseg > 0) {
      auto* cnt = reinterpret_cast<unsigned long long*>(h->hoff);
      const unsigned g = grid_for(sv.rows, 8, (int64_t)h->num_sms * 32);
      ++h->nlaunch;
      k_head_count<<<g, 256, 0, h->stream>>>(sv.T.ptr, h->nh, sv.T.ent, sv.rows, h->headslot, h->head_nd, nsp, cnt);
      launch_scan_inplace(h, h->hoff, nseg + 1, h->alloc<int64_t>(1));  // hoff[nseg] = total
      int64_t nhe = 0;
      CK(cudaMemcpyAsync(&nhe, h->hoff + nseg, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      h->hseg = h->alloc<int2>(std::max<int64_t>(nhe, 1));
      auto* cursor = static_cast<unsigned long long*>(h->tmp_get(sizeof(int64_t) * (nseg + 1)));
      CK(cudaMemcpyAsync(cursor, h->hoff, sizeof(int64_t) * (nseg + 1), cudaMemcpyDeviceToDevice, h->stream));
      ++h->nlaunch;
      k_head_fill<<<g, 256, 0, h->stream>>>(sv.T.ptr, h->nh, sv.T.ent, sv.rows, h->headslot, h->head_nd, nsp, cursor,
                                           h->hseg);
      h->tmp_put(cursor);
    } else {
      h->hseg = h->alloc<int2>(1);
    }
  }
  if (h->ptail) {  // paper-order tail: per-tile jagged-diagonal tail entries, Y_tail tiles, W', U row view
    const int64_t nt = h->head_ntiles;
    h->nyc = (h->kn + kHeadK - 1) / kHeadK;
    h->toff = h->alloc<int64_t>(nt + 1);
    CK(cudaMemsetAsync(h->toff, 0, sizeof(int64_t) * (nt + 1), h->stream));
    ++h->nlaunch;
    k_vt_count<<<(unsigned)nt, kVtM, 0, h->stream>>>(sv.T.ptr, hh > 0 ? h->nh : nullptr, sv.rows, h->toff);
    launch_scan_inplace(h, h->toff, nt + 1, h->alloc<int64_t>(1));
    int64_t ntail = 0;
    CK(cudaMemcpyAsync(&ntail, h->toff + nt, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->tent = h->alloc<int2>(std::max<int64_t>(ntail, 1));
    ++h->nlaunch;
    k_vt_fill<<<(unsigned)nt, kVtM, 0, h->stream>>>(sv.T.ptr, hh > 0 ? h->nh : nullptr, sv.T.ent, sv.rows, h->toff,
                                                   h->tent);
    if (ntail > 0 && ntail < (1LL << 31)) {  // sort every tile's entries by (term, row)
      auto* k0 = static_cast<uint32_t*>(h->tmp_get(sizeof(uint32_t) * ntail));
      auto* k1 = static_cast<uint32_t*>(h->tmp_get(sizeof(uint32_t) * ntail));
      auto* v0 = static_cast<int32_t*>(h->tmp_get(sizeof(int32_t) * ntail));
      auto* v1 = static_cast<int32_t*>(h->tmp_get(sizeof(int32_t) * ntail));
      const unsigned g = grid_for(ntail, 256, (int64_t)h->num_sms * 16);
      ++h->nlaunch;
      k_vt_to_keys<<<g, 256, 0, h->stream>>>(h->tent, ntail, k0, v0);
      int end_bit = 7;
      while (end_bit < 31 && (1LL << (end_bit - 7)) < n) ++end_bit;
      size_t tmp_bytes = 0;
      CK(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, v0, v1, (int)ntail, (int)nt, h->toff,
                                                  h->toff + 1, 0, end_bit, h->stream));
      void* tmp = h->tmp_get(tmp_bytes);
      CK(cub::DeviceSegmentedRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, (int)ntail, (int)nt, h->toff,
                                                  h->toff + 1, 0, end_bit, h->stream));
      ++h->nlaunch;
      k_vt_from_keys<<<g, 256, 0, h->stream>>>(k1, v1, ntail, h->tent);
      for (void* q : {(void*)k0, (void*)k1, (void*)v0, (void*)v1, tmp}) h->tmp_put(q);
    }
    h->ytile = h->alloc<uint8_t>(nt * kVtM * h->kn * 4);
    const int64_t wb = (int64_t)h->nyc * h->kn * kHeadK * 4;
    h->wbuf = h->alloc<uint8_t>(wb);
    CK(cudaMemsetAsync(h->wbuf, 0, wb, h->stream));
    h->umap = h->alloc<uint64_t>(n);
    CK(cudaMemsetAsync(h->umap, 0, sizeof(uint64_t) * n, h->stream));
    h->ubits = h->alloc<uint32_t>(ceil_div(n, 32));
    CK(cudaMemsetAsync(h->ubits, 0, sizeof(uint32_t) * ceil_div(n, 32), h->stream));
    h->vt_next = h->alloc<unsigned long long>(1);
    h->uent = h->alloc<int2>(n * (int64_t)(h->k + 1));  // rows padded to an even length
    h->urptr = h->alloc<int64_t>(n + 1);
    h->ucursor = h->alloc<int64_t>(n + 1);
    h->uscan = h->alloc<int64_t>(ceil_div(n + 1, kScanBlock) + 1);
    h->ulist = h->alloc<int32_t>(n);
    h->ulist_n = h->alloc<int64_t>(1);
    CK(cudaMemsetAsync(h->ulist_n, 0, sizeof(int64_t), h->stream));
    h->umax = h->alloc<uint32_t>(h->k);
    h->ushift = h->alloc<int>(h->k);
    h->Z64 = h->alloc<double>(n * (int64_t)h->k);
    if (const char* e = getenv("ESNMF_VT_KMAX")) h->vt_kmax = atof(e);
    if (const char* e = getenv("ESNMF_VT_AMAX")) h->vt_amax = atof(e);
    if (const char* e = getenv("ESNMF_VT_RATIO")) h->vt_ratio = atof(e);
    {
      std::vector<int32_t> tl(n);
      for (int64_t i = 0; i < n; ++i) tl[i] = (int32_t)(hptr[i + 1] - hptr[i]);
      h->termlen = h->alloc<int32_t>(n);
      CK(cudaMemcpyAsync(h->termlen, tl.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
    h->vcost = h->alloc<double>(8);
    CK(cudaMemsetAsync(h->vcost, 0, sizeof(double) * 8, h->stream));
    h->vt_ticket = h->alloc<unsigned>(1);
    CK(cudaMemsetAsync(h->vt_ticket, 0, sizeof(unsigned), h->stream));
    { const char* np_ = getenv("ESNMF_NO_POLISH"); h->polish = !(np_ && atoi(np_)); }
  }
  CKL("head_setup");
  // host vectors die here: make the async uploads complete first
  CK(cudaStreamSynchronize(h->stream));
}

// ---- paper-order V-side tail (k_vtail.cuh) ----
// U row view of the factor the V side reads: umap / uent (values scaled by 2^s_c)
void urows_build(esnmf_t* h, const Factor& f) {
  const int64_t nr = f.cap_rows + 1;
  h->nlaunch += 1;
  k_urows_clear<<<grid_for(f.cap_rows, 256, 4096), 256, 0, h->stream>>>(h->ulist, h->ulist_n, h->umap, h->ubits,
                                                                        h->vcost);
  CK(cudaMemsetAsync(h->urptr, 0, sizeof(int64_t) * nr, h->stream));
  dim3 g(col_grid_x(f.maxcol), h->k);
  ++h->nlaunch;
  k_vrows_count<<<g, 256, 0, h->stream>>>(f.colptr, f.row, f.rowmap, h->urptr);
  const int64_t nb = ceil_div(nr, kScanBlock);
  h->nlaunch += 3;
  // rows at even offsets (counts rounded up to even): k_ytail loads two pairs at a time
  k_blocksum_i64<<<(unsigned)nb, 256, 0, h->stream>>>(h->urptr, nr, h->uscan, 1);
  k_scan_small<<<1, 1024, 0, h->stream>>>(h->uscan, nb, h->uscan + nb);
  k_scan_apply_i64<<<(unsigned)nb, 256, 0, h->stream>>>(h->urptr, nr, h->uscan, 1);
  CK(cudaMemcpyAsync(h->ucursor, h->urptr, sizeof(int64_t) * nr, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaMemsetAsync(h->umax, 0, sizeof(uint32_t) * h->k, h->stream));
  h->nlaunch += 3;
  k_urows_scatter<<<g, 256, 0, h->stream>>>(f.colptr, f.row, f.val, f.rowmap, h->head_h > 0 ? h->headslot : nullptr,
                                            h->ucursor, h->uent, h->umax);
  // (every slot up to the padded total, uscan[nb]; the pads, written next, are skipped)
  k_ut_scale<<<grid_for(f.cap, 256, (int64_t)h->num_sms * 8), 256, 0, h->stream>>>(h->uscan + nb, h->uent, h->k,
                                                                                   h->umax, h->rowsum_bits, h->ushift);
  k_urows_finish<<<grid_for(f.cap_rows, 256, 4096), 256, 0, h->stream>>>(
      f.active, f.n_active, h->urptr, h->ucursor, h->uent, h->umap, h->ubits, h->ulist, h->ulist_n, h->termlen,
      h->head_h > 0 ? h->headslot : nullptr, h->k, h->vcost, h->vt_ticket, h->vt_ratio, h->flags + 5);
  CKL("urows_build");
}

void ytail_launch(esnmf_t* h) {
  const int ys = h->kn | 1;
  const size_t smem = ytail_smem(ys);
  CK(cudaFuncSetAttribute(k_ytail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_ytail, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = std::max(1, std::min(kVtMinB, (int)((228 * 1024) / (smem + 1024))));
  if (const char* e = getenv("ESNMF_YTAIL_PERSM")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
  const unsigned grid = (unsigned)std::min<int64_t>(h->head_ntiles, (int64_t)h->num_sms * per_sm);
  CK(cudaMemsetAsync(h->vt_next, 0, sizeof(unsigned long long), h->stream));
  ++h->nlaunch;
  k_ytail<<<grid, kVtThreads, smem, h->stream>>>(h->toff, h->tent, h->head_ntiles, h->ubits, h->umap, h->uent, h->kn,
                                                  ys, h->ytile, h->vt_next, h->flags + 5);
  CKL("ytail");
}

// kept V entries recomputed exactly (k_polish_v); not with Alg. 3's deflation
void polish_v(esnmf_t* h, const int64_t* colptr, const int32_t* row, float* val) {
  if (!h->ptail || (h->ktot && h->seq_b > 0) || !h->polish) return;  // (Alg. 3 deflates later blocks' LS)
  Side& sv = h->side[ESNMF_SIDE_V];
  const int64_t per_col = h->tside[ESNMF_SIDE_V] < 0 ? sv.rows : std::min<int64_t>(h->tside[ESNMF_SIDE_V], sv.rows);
  const dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(per_col, 16), 4096)), h->k);  // 2 per warp
  ++h->nlaunch;
  k_polish_v<<<g, 256, 0, h->stream>>>(colptr, row, val, h->k, sv.row0, sv.T.ptr, sv.T.ent, h->ubits, h->Z64);
  CKL("polish_v");
}

// kept U entries recomputed exactly from the fixed-point A V (one GPU; k_polish_u)
void polish_u(esnmf_t* h, Factor& out) {
  if (h->sharded || !h->Yq || !h->polish || (h->ktot && h->seq_b > 0)) return;
  const int64_t per_col = h->tside[ESNMF_SIDE_U] < 0 ? h->n : std::min<int64_t>(h->tside[ESNMF_SIDE_U], h->n);
  const dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(per_col, 16), 4096)), h->k);  // 2 per warp
  ++h->nlaunch;
  k_polish_u<<<g, 256, 0, h->stream>>>(out.colptr, out.row, out.val, h->k, h->kpad, h->Yq, h->rsum_max, h->vmax,
                                       h->W);
  CKL("polish_u");
}

// Z64 = U W for U's active rows (fp64; k_form_z64), term-indexed
void form_z64(esnmf_t* h, const Factor& f) {
  const unsigned grid = grid_for(f.cap_rows, 8, (int64_t)h->num_sms * 16);
  ++h->nlaunch;
  switch ((h->k + 31) / 32) {
    case 1: k_form_z64<1><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->W, h->Z64); break;
    case 2: k_form_z64<2><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->W, h->Z64); break;
    case 3: k_form_z64<3><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->W, h->Z64); break;
    case 4: k_form_z64<4><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->W, h->Z64); break;
    case 5: k_form_z64<5><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->W, h->Z64); break;
    case 6: k_form_z64<6><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->W, h->Z64); break;
    case 7: k_form_z64<7><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->W, h->Z64); break;
    default: k_form_z64<8><<<grid, 256, 0, h->stream>>>(f.dense, h->kpad, h->k, f.n_active, f.active, h->W, h->Z64); break;
  }
  CKL("form_z64");
}

void vside_prep(esnmf_t* h, const Factor& f) {
  ++h->nlaunch;
  k_vside_prep<<<h->k, 256, 0, h->stream>>>(h->Z64, f.rowmap, h->headterm, h->head_h, h->W, h->k, h->kn,
                                            h->amax_bits, h->ushift, h->zhead, h->wbuf, h->colscale, h->flags + 4);
  CKL("vside_prep");
}

// U-side fixed-point accumulator: the U side uses Yqb[ucur]; the V side after it
// clears the other buffer (the one the previous U side used and k_polish_u read)
void yq_clear_other(esnmf_t* h) {
  if (!h->Yqb[0] || !h->yq_other_dirty) return;
  CK(cudaMemsetAsync(h->Yqb[1 - h->yq_par], 0, sizeof(unsigned long long) * h->n * h->kpad, h->stream));
  h->yq_other_dirty = false;
}

// the V side's operands after the solve: Z = U W (fp64; the head's Z chunks and the
// exact kept values), the Z-row gather (the paper-order tail's fallback: its kernels
// return at once otherwise) and the head's operand prep
// (gather_aux: the gather's launches on aux beside the prep)
void vside_ops(esnmf_t* h, const Factor& in, bool gather_aux) {
  form_z64(h, in);
  if (gather_aux) fork_to_aux(h, h->ev_vfork);
  {
    OnStream os(h, gather_aux ? h->aux : h->stream);
    Phase ph(h, kVGather);
    form_z(h, in, h->flags + 4);
    spmm(h, ESNMF_SIDE_V, in.rowmap, h->flags + 4);
  }
  { Phase ph(h, kVFormZ); vside_prep(h, in); }
  if (gather_aux) join_from_aux(h, h->ev_vjoin);
}

// one half-step; returns the factor that was written
Factor& half_step(esnmf_t* h, int s) {
  Side& sd = h->side[s];
  Factor& in = (s == ESNMF_SIDE_V) ? h->U[h->ucur] : h->V;
  Factor& out = (s == ESNMF_SIDE_V) ? h->V : h->U[1 - h->ucur];
  if (!in.has) fail(ESNMF_ESTATE, s == ESNMF_SIDE_V ? "U is not set" : "V is not set (run the V side first)");
  const int p0 = s == ESNMF_SIDE_V ? kVGram : kUGram;
  const bool overlap_u = s == ESNMF_SIDE_U && !h->sharded;    // Gram + solve on aux, beside the scatter
  if (s == ESNMF_SIDE_U) join_metrics(h);  // (only pending after a bare half_step call)
  if (s == ESNMF_SIDE_U && h->Yqb[0]) {
    h->Yq = h->Yqb[h->yq_par];
    if (!h->v_since_u)  // two U sides in a row (bare half_step calls): this buffer is the dirty one
      CK(cudaMemsetAsync(h->Yq, 0, sizeof(unsigned long long) * h->n * h->kpad, h->stream));
    h->v_since_u = false;
  }
  if (s == ESNMF_SIDE_V) h->v_since_u = true;
  if (h->gram_on_aux) {  // G_U on aux: only the paper-order V side's solve (on aux) is ordered after it
    const bool solve_on_aux = s == ESNMF_SIDE_V && h->ptail && !getenv("ESNMF_V_SERIAL");
    if (!solve_on_aux) join_from_aux(h, h->ev_gjoin);
    h->gram_on_aux = false;
  }
  if (s == ESNMF_SIDE_V && h->ptail) {
    // paper-order tail (k_vtail.cuh): Y_tail = A^T_tail U needs only U, so the
    // Gram + solve (a1, a2) run on aux beside it; then Z_head = U_head W, the
    // scales, and the tensor-core kernel: head chunks + (Y_tail W) chunks
    {
      Phase ph(h, kVFormZ);
      // + the cost model: paper order or Z-row gather for the tail this time
      urows_build(h, in);
    }
    const bool vser = getenv("ESNMF_V_SERIAL") != nullptr;  // (measurement: the solve before the tail, one stream)
    static const bool prep_aux = getenv("ESNMF_VPREP_MAIN") == nullptr;
    if (!vser) fork_to_aux(h, h->ev_vfork);
    {
      OnStream os(h, vser ? h->stream : h->aux);
      if (!h->gramU_valid) { Phase ph(h, p0 + 0); gram(h, in, sd.G); }   // a1: P:63
      {  // a2, and: is Y_tail W safe in fp16 hi/lo this time?  (else: Z-row gather; flags[4])
        Phase ph(h, p0 + 1);
        SweepCond sc;
        sc.flag = h->flags + 4;
        sc.kmax = h->vt_kmax;
        sc.amax = h->vt_amax;
        sc.orflag = h->flags + 5;
        sweep(h, sd.G, sd.eps, sc);
      }
      // everything else the head needs depends on U and W only, so it follows the
      // solve on aux beside the tail product instead of between the tail and the
      // head: Z = U W (fp64; the head's Z chunks and the exact kept values), the
      // Z-row gather (fallback only: its kernels return at once otherwise) and the
      // head's operand prep
      if (prep_aux) vside_ops(h, in, false);
    }
    { Phase ph(h, kVSpmm); ytail_launch(h); }                             // a3 (tail, paper order)
    if (!vser) join_from_aux(h, h->ev_vjoin);
    if (!prep_aux) vside_ops(h, in, !vser);
    { Phase ph(h, kVHead); vhead_launch(h, false); }                      // a3 + a4 (head, tail x W)
    if (getenv("ESNMF_DEBUG_VT")) {
      CK(cudaStreamSynchronize(h->stream));
      int fl[8];
      CK(cudaMemcpy(fl, h->flags, sizeof(fl), cudaMemcpyDeviceToHost));
      std::vector<float> xt(std::min<int64_t>(sd.rows * h->kpad, 4096)), x(std::min<int64_t>(sd.ldx * h->k, 4096));
      CK(cudaMemcpy(xt.data(), sd.Xt, sizeof(float) * xt.size(), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(x.data(), sd.X, sizeof(float) * x.size(), cudaMemcpyDeviceToHost));
      double a = 0, b = 0;
      for (float v : xt) a += fabs(v);
      for (float v : x) b += fabs(v);
      fprintf(stderr, "ESNMF_DEBUG_VT flag4=%d |Xt|=%g |X|=%g head=%d nyc=%d\n", fl[4], a, b, h->head_h, h->nyc);
    }
  } else if (!(overlap_u && h->u_prefork)) {
    if (overlap_u) fork_to_aux(h, h->ev_ufork);
    OnStream os(h, overlap_u ? h->aux : h->stream);
    if (!(s == ESNMF_SIDE_V && h->gramU_valid)) {                 // a1: P:63 / P:64
      Phase ph(h, p0 + 0);
      gram(h, in, sd.G);
    }
    {  // a2 (U side: is the fp32 / tensor-core (Y W) safe?  flags[3])
      Phase ph(h, p0 + 1);
      SweepCond sc;
      if (s == ESNMF_SIDE_U) sc.flag = h->flags + 3, sc.kmax = h->u_kmax;
      sweep(h, sd.G, sd.eps, sc);
    }
    if (overlap_u) uside_w_prep(h);
  }
  h->u_prefork = false;
  if (!(s == ESNMF_SIDE_V && h->ptail)) {
    if (s == ESNMF_SIDE_V) { Phase ph(h, p0 + 2); form_z(h, in); }   // Z = U W (V side only)
    { Phase ph(h, p0 + 3); spmm(h, s, in.rowmap); }                  // a3 (+a4 scale); V: tail terms
    if (s == ESNMF_SIDE_V && h->head_h > 0) { Phase ph(h, kVHead); vhead_launch(h, false); }  // V: head terms (TC)
  }
  seq_deflate(h, s);                                               // Alg. 3: Eq. (7) / (8)
  sd.ls_valid = true;
  {
    Phase ph(h, p0 + 4);
    join_metrics(h);  // the previous iteration's record reads V
    if (s == ESNMF_SIDE_V) vrows_clear(h);
    factor_clear(h, out);
    if (!h->sharded) {
      select_topt(h, s, out);                                      // a4 clamp + a5 top-t
      if (s == ESNMF_SIDE_V) polish_v(h, out.colptr, out.row, out.val);
      else polish_u(h, out);
    } else {
      select_merge(h, s, out);                                     // + a6 shard merge
    }
  }
  {
    Phase ph(h, p0 + 5);
    factor_build_rows(h, out, steady_maxcol(h, s, out.rows));
    if (s == ESNMF_SIDE_V && !h->sharded) {
      // the U side's a1 + a2 need only V's row view: start them now on aux,
      // beside V's row-CSR build and the U side's scatter
      fork_to_aux(h, h->ev_ufork);
      OnStream os(h, h->aux);
      Side& su = h->side[ESNMF_SIDE_U];
      { Phase ph2(h, kUGram); gram(h, out, su.G); }
      if (!need_vrows(h)) CK(cudaEventRecord(h->ev_ugram, h->stream));
      {
        Phase ph2(h, kUSolve);
        SweepCond sc;
        sc.flag = h->flags + 3;
        sc.kmax = h->u_kmax;
        sweep(h, su.G, su.eps, sc);
      }
      yq_clear_other(h);  // the buffer the last U side used, unless the record cleared it
      uside_w_prep(h);
      h->u_prefork = true;
    }
    if (s == ESNMF_SIDE_V) {
      vrows_build(h);
      if (!h->sharded && !need_vrows(h)) CK(cudaStreamWaitEvent(h->stream, h->ev_ugram, 0));
    }
  }
  if (s == ESNMF_SIDE_U) {
    h->ucur = 1 - h->ucur;
    h->yq_par = 1 - h->yq_par;
    if (h->Yqb[0]) h->yq_other_dirty = true;
    h->gramU_valid = false;
  }
  return out;
}

void ensure_records(esnmf_t* h, int64_t need) {
  if (need <= h->rec_cap) return;
  int64_t cap = std::max<int64_t>(need, 2 * h->rec_cap + 64);
  esnmf_record* r = h->alloc<esnmf_record>(cap);
  if (h->nrec > 0) CK(cudaMemcpyAsync(r, h->rec, sizeof(esnmf_record) * h->nrec, cudaMemcpyDeviceToDevice, h->stream));
  h->rec = r;
  h->rec_cap = cap;
}

void flush_metrics(esnmf_t* h);

// One iteration.  Its R / E record (a7, a8) is launched at the start of the
// next iteration (or by esnmf_iterate's final flush): the same stream order as
// launching it at the end, but every iteration is then a self-contained unit
// for CUDA-graph capture (the record's aux-stream kernels are joined inside the
// next V side).
void iterate_one(esnmf_t* h) {
  flush_metrics(h);
  if (h->ktot && h->seq_i == h->seq_iters) {
    if ((h->seq_b + 1) * h->seq_k2 >= h->ktot) fail(ESNMF_ESTATE, "sequential ALS: all k / k2 blocks are done");
    seq_next_block(h);
  }
  half_step(h, ESNMF_SIDE_V);
  half_step(h, ESNMF_SIDE_U);
  h->metrics_pending = true;
  if (h->ktot) ++h->seq_i;  // after seq_iters: the next iterate appends the block (seq_next_block)
}

// R, E and the record of the last iteration, and the Gram of its U
void flush_metrics(esnmf_t* h) {
  if (!h->metrics_pending) return;
  h->metrics_pending = false;
  Phase ph(h, kMetrics);
  Factor& Un = h->U[h->ucur];
  Factor& Uo = h->U[1 - h->ucur];
  const int k = h->k;
  // a7 residual, direct difference
  const unsigned gxn = col_grid_x(Un.maxcol), gxo = col_grid_x(Uo.maxcol);
  double* p_new = h->red;
  double* p_old = p_new + 2 * (int64_t)gxn * k;
  double* p_tr = p_old + (int64_t)gxo * k;
  // Gram of the new U first (the next V side's solve waits for it): S term of E, G_U.
  // On one GPU it runs on aux (ahead of that solve, beside the next V side's U row
  // view on main) and the record's stream starts after it.
  const bool overlap_m = !h->sharded;
  if (overlap_m) {
    fork_to(h, h->aux, h->ev_gfork);
    OnStream og(h, h->aux);
    gram(h, Un, h->side[ESNMF_SIDE_V].G);
    fork_to(h, h->maux, h->ev_mfork);  // maux: after main's state (via aux) and the Gram
    h->gram_on_aux = true;
  } else {
    gram(h, Un, h->side[ESNMF_SIDE_V].G);
  }
  h->gramU_valid = true;
  // a8 error: T = tr(U^T (A V)) from the U side's LS rows.  On one GPU
  // the trace and the record run on the aux stream, beside the next V side
  // (joined before that V side replaces V, join_metrics).
  OnStream os(h, overlap_m ? h->maux : h->stream);
  // (on the aux stream: U_{i-1} is overwritten only by the next U side, after the join)
  ++h->nlaunch; k_resid_new<<<dim3(gxn, k), 256, 0, h->stream>>>(Un.colptr, Un.row, Un.val, Uo.rowmap, Uo.dense, h->kpad, p_new);
  ++h->nlaunch; k_resid_old<<<dim3(gxo, k), 256, 0, h->stream>>>(Uo.colptr, Uo.row, Uo.val, Un.rowmap, Un.dense, h->kpad, p_old);
  Side& su = h->side[ESNMF_SIDE_U];
  const unsigned gtr = grid_for(Un.cap_rows, 8, (int64_t)h->num_sms * 8);
  ++h->nlaunch;
#define ESNMF_ET(cq)                                                                                              \
  case cq:                                                                                                        \
    k_err_trace_rows<cq><<<gtr, 256, 0, h->stream>>>(Un.active, Un.n_active, Un.dense, h->kpad, su.row0, su.rows, \
                                                     su.X, su.ldx, su.G, su.eps, k, p_tr);                        \
    break;
  switch ((k + 31) / 32) {
    ESNMF_ET(1) ESNMF_ET(2) ESNMF_ET(3) ESNMF_ET(4) ESNMF_ET(5) ESNMF_ET(6) ESNMF_ET(7)
    default: k_err_trace_rows<8><<<gtr, 256, 0, h->stream>>>(Un.active, Un.n_active, Un.dense, h->kpad, su.row0,
                                                             su.rows, su.X, su.ldx, su.G, su.eps, k, p_tr);
  }
#undef ESNMF_ET
  CKL("metrics");
  const double* t_red = nullptr;
  if (h->sharded) {
    ++h->nlaunch;
    k_rank_scalars<<<1, 256, 0, h->stream>>>(p_tr, (int64_t)gtr, su.peak, h->side[ESNMF_SIDE_V].peak, h->scal + 3);
    if (h->comm.allreduce_sum_f64(h->comm.ctx, h->scal + 3, 3, h->stream) != 0)
      fail(ESNMF_ECOMM, "allreduce(T, peaks) failed");
    t_red = h->scal + 3;
  }
  ensure_records(h, h->nrec + 1);
  RecordInputs in;
  in.rnew = p_new;
  in.nrnew = (int64_t)gxn * k;
  in.rold = p_old;
  in.nrold = (int64_t)gxo * k;
  in.tpart = p_tr;
  in.ntpart = (int64_t)gtr;
  in.GU = h->side[ESNMF_SIDE_V].G;
  in.GV = su.G;
  in.colptr_u = Un.colptr;
  in.colptr_v = h->V.colptr;
  in.nact_u = Un.n_active;
  in.nact_v = h->V.n_active;
  in.peak_u = su.peak;
  in.peak_v = h->side[ESNMF_SIDE_V].peak;
  in.normA2 = h->normA2;
  in.k = k;
  in.t_reduced = t_red;
  if (h->ktot) {  // whole-factor records: the converged columns' constant terms
    in.seqc = h->seqc;
    in.fcolptr_u = h->FU.colptr;
    in.fcolptr_v = h->FV.colptr;
    in.ktot = h->ktot;
    in.b0 = h->seq_b * h->seq_k2;
  }
  ++h->nlaunch; k_finalize_record<<<1, 256, 0, h->stream>>>(in, h->rec, h->d_nrec, h->scal);
  CKL("finalize_record");
  // the last U side's fixed-point buffer (k_polish_u has read it) is cleared here, on
  // the low-priority stream beside the next V side, instead of on the aux stream
  // ahead of the next U side's W preparation (n x kpad x 8 bytes: 166 MB at Large)
  if (overlap_m) yq_clear_other(h);
  h->nrec += 1;
  if (overlap_m) h->aux_pending = true;
}

// ---- CUDA graphs of the steady-state iteration ----
void graph_reset(esnmf_t* h) {
  for (int p = 0; p < 2; ++p)
    if (h->gexec[p]) {
      cudaGraphExecDestroy(h->gexec[p]);
      h->gexec[p] = nullptr;
    }
  h->steady = 0;
}

// two eager iterations since the last state change: every host-side launch
// parameter (factor column bounds, selection paths, record slot base) is then
// the same in every later iteration.  Single GPU, profiling off; in sequential
// ALS within a block (a block change runs eagerly and drops the graphs).
bool graph_ok(esnmf_t* h) {
  return !getenv("ESNMF_NO_GRAPH") && (!h->sharded || builtin_nccl(h->comm)) && !h->prof_on && h->steady >= 2 && h->metrics_pending &&
         !h->u_prefork && !h->aux_pending && !(h->ktot && h->seq_i >= h->seq_iters);
}

// one iteration (with the previous one's record) as one graph launch; one graph
// per U slot parity (the iteration reads U[ucur] and writes U[1 - ucur]).  The
// first call per parity captures it (running iterate_one, which advances the
// host state exactly as a replay does) and launches it.
void graph_run(esnmf_t* h) {
  const int p = h->ucur;
  if (h->gexec[p] && h->grec[p] != h->rec) {
    cudaGraphExecDestroy(h->gexec[p]);
    h->gexec[p] = nullptr;
  }
  if (!h->gexec[p]) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
    const int64_t l0 = h->nlaunch;
    try {
      iterate_one(h);
      if (h->aux_pending || h->u_prefork) fail(ESNMF_ECUDA, "graph capture: unjoined aux-stream work");
    } catch (...) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(h->stream, &junk);
      if (junk) cudaGraphDestroy(junk);
      throw;
    }
    CK(cudaStreamEndCapture(h->stream, &g));
    const cudaError_t e = cudaGraphInstantiate(&h->gexec[p], g, 0);
    cudaGraphDestroy(g);
    CK(e);
    h->grec[p] = h->rec;
    h->glaunch[p] = h->nlaunch - l0;
    CK(cudaGraphLaunch(h->gexec[p], h->stream));
    return;
  }
  CK(cudaGraphLaunch(h->gexec[p], h->stream));
  h->nlaunch += h->glaunch[p];
  h->nrec += 1;       // the previous iteration's record (device slot counter d_nrec advanced by the graph)
  h->ucur = 1 - h->ucur;
  h->yq_par = 1 - h->yq_par;
  h->gramU_valid = false;
  h->metrics_pending = true;
  if (h->ktot) ++h->seq_i;
}

void sync_check(esnmf_t* h) {
  CK(cudaStreamSynchronize(h->stream));
  int fl[3];
  CK(cudaMemcpy(fl, h->flags, sizeof(fl), cudaMemcpyDeviceToHost));
  if (fl[0]) fail(ESNMF_ESINGULAR, "G + eps I is not positive definite (non-positive or non-finite pivot)");
}

// U side work items over this shard's term rows (host, from a copy of row_ptr)
void build_items(esnmf_t* h, Side& sd, const std::vector<int64_t>& ptr_local) {
  std::vector<WorkItem> items;
  std::vector<int32_t> slot;
  std::vector<SplitRow> splits;
  int64_t nslots = 0;
  for (int64_t r = 0; r < sd.rows; ++r) {
    const int64_t s = ptr_local[r], e = ptr_local[r + 1], len = e - s;
    const int64_t nit = std::max<int64_t>(1, ceil_div(len, kSplitLen));
    if (nit == 1) {
      items.push_back(WorkItem{s, (int32_t)r, (int32_t)len});
      slot.push_back(-1);
    } else {
      splits.push_back(SplitRow{(int32_t)r, (int32_t)nslots, (int32_t)nit, 0});
      for (int64_t q = 0; q < nit; ++q) {
        const int64_t b = s + q * kSplitLen;
        items.push_back(WorkItem{b, (int32_t)r, (int32_t)std::min<int64_t>(kSplitLen, e - b)});
        slot.push_back((int32_t)nslots++);
      }
    }
  }
  sd.nitems = (int64_t)items.size();
  sd.nsplit = (int64_t)splits.size();
  sd.nslots = nslots;
  sd.items = h->alloc<WorkItem>(sd.nitems);
  sd.item_slot = h->alloc<int32_t>(sd.nitems);
  sd.splits = h->alloc<SplitRow>(sd.nsplit);
  sd.partial = reinterpret_cast<float*>(h->alloc<unsigned long long>(std::max<int64_t>(1, nslots) * h->kpad));
  CK(cudaMemcpy(sd.items, items.data(), sizeof(WorkItem) * sd.nitems, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(sd.item_slot, slot.data(), sizeof(int32_t) * sd.nitems, cudaMemcpyHostToDevice));
  if (sd.nsplit) CK(cudaMemcpy(sd.splits, splits.data(), sizeof(SplitRow) * sd.nsplit, cudaMemcpyHostToDevice));
}

void side_alloc(esnmf_t* h, Side& sd) {
  const int k = h->k;
  sd.ldx = std::max<int64_t>(32, ceil_div(sd.rows, 32) * 32);
  sd.X = h->alloc<float>((int64_t)k * sd.ldx);
  CK(cudaMemsetAsync(sd.X, 0, sizeof(float) * k * sd.ldx, h->stream));  // padding rows stay 0 (flat view)
  sd.nchunks = std::max<int64_t>(1, ceil_div(sd.rows, kSelChunk));
  sd.hist = h->alloc<uint32_t>((int64_t)k * kNumBins);
  sd.sel = h->alloc<ColSel>(k);
  // threshold-bucket candidates per column: kSelCap are sorted on chip; with the
  // 3-pass path (t > kSelFastT or unlimited) a larger list keeps a big bucket
  // off the grid-wide radix passes over X (Box: each pass reads 6.4 GB)
  {
    const int64_t tt = h->tside[&sd == &h->side[ESNMF_SIDE_V] ? 0 : 1];
    sd.ccap = (tt < 0 || tt > kSelFastT) ? (int)std::min<int64_t>(65536, std::max<int64_t>(kSelCap, sd.rows / 16))
                                         : kSelCap;
  }
  sd.cand = h->alloc<uint64_t>((int64_t)k * sd.ccap);
  sd.cand_fill = h->alloc<int32_t>(k);
  sd.chunk_cnt = h->alloc<int64_t>((int64_t)k * (sd.nchunks + 1) * kSelSegs);  // (+1: the flat view)
  sd.coltot = h->alloc<int64_t>(k);
  sd.kthr = h->alloc<uint64_t>(k);
  sd.lvl = h->alloc<SelLvl>(k);
  sd.scanbuf = h->alloc<int64_t>(kSelScanMax);
  const int64_t ts = h->tside[&sd == &h->side[ESNMF_SIDE_V] ? 0 : 1];
  if (ts >= 0 && ts <= kSelFastT) {
    sd.above = h->alloc<uint64_t>((int64_t)k * std::max<int64_t>(ts, 1));
    sd.above_t = std::max<int64_t>(ts, 1);
    sd.above_fill = h->alloc<int32_t>(2 * (int64_t)k);
    sd.bucket = h->alloc<uint64_t>((int64_t)k * kSelCap);
    // predicted-threshold single pass: worth its extra kernel when the LS buffer is
    // large (Large: V side 400 MB, U side 80 MB: U.select 0.131 -> 0.124 ms)
    int64_t min_rows = 1 << 17;
    if (const char* pe = getenv("ESNMF_PRED_MIN_ROWS")) min_rows = atoll(pe);  // tests force it on small shards
    if (sd.rows >= min_rows) {
      sd.pcap = (int)std::min<int64_t>(kPredSort, 2 * ts + 2048);
      sd.pred = h->alloc<uint32_t>(k);
      CK(cudaMemsetAsync(sd.pred, 0xFF, sizeof(uint32_t) * k, h->stream));
      sd.pcand = h->alloc<uint64_t>((int64_t)k * sd.pcap);
      sd.pfill = h->alloc<int32_t>(2 * (int64_t)k);
      sd.npos = h->alloc<int32_t>(k);
    }
  }
  sd.G = h->alloc<double>((int64_t)k * k);
  sd.peak = h->alloc<int64_t>(1);
  CK(cudaMemsetAsync(sd.peak, 0, sizeof(int64_t), h->stream));
  sd.eps = h->alloc<double>(1);
  if (h->sharded) {
    const int64_t rows_max = (&sd == &h->side[ESNMF_SIDE_V]) ? h->v_rows_max : h->u_rows_max;
    sd.cap_s = std::max<int64_t>(1, ts < 0 ? rows_max : std::min(ts, rows_max));
    sd.lcolptr = h->alloc<int64_t>(k + 1);
    sd.lrow = h->alloc<int32_t>((int64_t)k * sd.cap_s);
    sd.lval = h->alloc<float>((int64_t)k * sd.cap_s);
    sd.shard_bytes = shard_bytes(k, sd.cap_s);
    sd.sendbuf = h->alloc<unsigned char>((int64_t)sd.shard_bytes);
    sd.recvbuf = h->alloc<unsigned char>((int64_t)sd.shard_bytes * h->world);
    sd.mscratch = h->alloc<uint64_t>((int64_t)k * 2 * sd.cap_s * h->world);
  }
}

// multi-rank clamp + top-t: local selection over this rank's rows, allgather
// of the candidates, identical deterministic merge on every rank (k_merge.cuh)
void select_topt(esnmf_t* h, int s, Factor& out);
void select_merge(esnmf_t* h, int s, Factor& out) {
  Side& sd = h->side[s];
  const int k = h->k;
  Factor loc;
  loc.colptr = sd.lcolptr;
  loc.row = sd.lrow;
  loc.val = sd.lval;
  select_topt(h, s, loc);
  if (s == ESNMF_SIDE_V) polish_v(h, loc.colptr, loc.row, loc.val);  // exact values before the exchange
  dim3 g(col_grid_x(sd.cap_s), k);
  ++h->nlaunch;
  k_pack_shard<<<g, 256, 0, h->stream>>>(sd.lcolptr, sd.lrow, sd.lval, k, sd.cap_s, sd.sendbuf);
  CKL("pack_shard");
  if (h->comm.allgather(h->comm.ctx, sd.sendbuf, sd.recvbuf, (int64_t)sd.shard_bytes, h->stream) != 0)
    fail(ESNMF_ECOMM, "allgather(top-t candidates) failed");
  h->nlaunch += 2;
  k_merge_counts<<<1, 256, 0, h->stream>>>(sd.recvbuf, sd.shard_bytes, h->world, k, sd.cap_s, h->tside[s],
                                           out.colptr);
  k_merge_topt<<<k, 1024, 0, h->stream>>>(sd.recvbuf, sd.shard_bytes, h->world, k, sd.cap_s, h->tside[s], out.colptr,
                                          out.row, out.val, sd.mscratch);
  CKL("merge_topt");
}

// upload (or copy) a CSR and pack it; returns device CSR with local rows [r0, r1)
// balanced create-time work units over a CSR's rows (host row pointers, local)
RowChunk* make_chunks(esnmf_t* h, const std::vector<int64_t>& lp, int64_t rows, int64_t* nch_out) {
  std::vector<RowChunk> v;
  v.reserve(rows + (lp[rows] / kChunkLen) + 1);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t b = lp[r]; b < lp[r + 1]; b += kChunkLen) v.push_back(RowChunk{b, std::min(lp[r + 1], b + kChunkLen), (int32_t)r, 0});
  *nch_out = (int64_t)v.size();
  RowChunk* d = h->alloc<RowChunk>(std::max<int64_t>(1, (int64_t)v.size()));
  if (!v.empty()) CK(cudaMemcpy(d, v.data(), sizeof(RowChunk) * v.size(), cudaMemcpyHostToDevice));
  return d;
}

DevCsr upload_csr(esnmf_t* h, int64_t rows_total, int64_t cols, const int64_t* ptr, const int32_t* col,
                  const float* val, bool on_dev, int64_t r0, int64_t r1, std::vector<int64_t>* host_ptr_local) {
  DevCsr c;
  c.rows = r1 - r0;
  c.cols = cols;
  std::vector<int64_t> hp(rows_total + 1);
  CK(cudaMemcpy(hp.data(), ptr, sizeof(int64_t) * (rows_total + 1), on_dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
  if (hp[0] != 0) fail(ESNMF_EINVAL, "row_ptr[0] != 0");
  for (int64_t r = 0; r < rows_total; ++r)
    if (hp[r + 1] < hp[r]) fail(ESNMF_EINVAL, "row_ptr is not non-decreasing at row " + std::to_string(r));
  const int64_t e0 = hp[r0], e1 = hp[r1];
  c.nnz = e1 - e0;
  c.ptr = h->alloc<int64_t>(c.rows + 1);
  std::vector<int64_t> lp(c.rows + 1);
  for (int64_t r = 0; r <= c.rows; ++r) lp[r] = hp[r0 + r] - e0;
  CK(cudaMemcpy(c.ptr, lp.data(), sizeof(int64_t) * (c.rows + 1), cudaMemcpyHostToDevice));
  c.ent = h->alloc<int2>(c.nnz);
  if (c.nnz > 0) {
    int32_t* dcol;
    float* dval;
    if (on_dev) {
      dcol = const_cast<int32_t*>(col) + e0;
      dval = const_cast<float*>(val) + e0;
    } else {
      // stage through the (not yet used) entry buffer's tail: pack from two temporaries
      dcol = h->alloc<int32_t>(c.nnz);
      dval = h->alloc<float>(c.nnz);
      CK(cudaMemcpyAsync(dcol, col + e0, sizeof(int32_t) * c.nnz, cudaMemcpyHostToDevice, h->stream));
      CK(cudaMemcpyAsync(dval, val + e0, sizeof(float) * c.nnz, cudaMemcpyHostToDevice, h->stream));
    }
    ++h->nlaunch; k_pack<<<grid_for(c.nnz, 256, 148 * 32), 256, 0, h->stream>>>(dcol, dval, c.nnz, c.ent);
    CKL("pack");
    if (!on_dev) {
      CK(cudaStreamSynchronize(h->stream));
      // release the staging buffers now (they were the last two allocations)
      for (int q = 0; q < 2; ++q) {
        void* p = h->allocs.back();
        h->allocs.pop_back();
        h->release(p);
      }
      h->bytes -= (int64_t)(sizeof(int32_t) + sizeof(float)) * c.nnz;
    }
  }
  {
    int64_t nch = 0;
    c.chunks = make_chunks(h, lp, c.rows, &nch);
    c.nchunks = nch;
    ++h->nlaunch;
    k_validate_chunks<<<grid_for(nch, 8, (int64_t)h->num_sms * 64), 256, 0, h->stream>>>(c.chunks, nch, c.ptr, c.ent,
                                                                                         cols, h->flags + 1);
  }
  CKL("validate");
  if (host_ptr_local) *host_ptr_local = std::move(lp);
  return c;
}

// CSR(A^T) rows [m0, m1) built on the device from the full CSR(A)
DevCsr build_at(esnmf_t* h, const DevCsr& A, int64_t m, int64_t m0, int64_t m1) {
  DevCsr T;
  T.rows = m;
  T.cols = A.rows;
  T.nnz = A.nnz;
  T.ptr = h->alloc<int64_t>(m + 1);
  T.ent = h->alloc<int2>(A.nnz);
  CK(cudaMemsetAsync(T.ptr, 0, sizeof(int64_t) * (m + 1), h->stream));
  ++h->nlaunch; k_col_count<<<grid_for(A.nnz, 256, 148 * 32), 256, 0, h->stream>>>(A.ent, A.nnz, T.ptr);
  int64_t* tot = h->alloc<int64_t>(1);
  launch_scan_inplace(h, T.ptr, m + 1, tot);
  int64_t* cursor = h->alloc<int64_t>(m + 1);
  CK(cudaMemcpyAsync(cursor, T.ptr, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToDevice, h->stream));
  if (!A.chunks) fail(ESNMF_EINVAL, "build_at: operator without work units");
  ++h->nlaunch;
  k_transpose_chunks<<<grid_for(A.nchunks, 8, (int64_t)h->num_sms * 64), 256, 0, h->stream>>>(
      A.chunks, A.nchunks, A.ent, reinterpret_cast<unsigned long long*>(cursor), T.ent);
  ++h->nlaunch;
  k_sort_rows_rank<<<grid_for(m, 8, (int64_t)h->num_sms * 32), 256, 0, h->stream>>>(T.ptr, m, T.ent);
  // long rows (> kRowSortCap entries) in a global scratch, one block
  std::vector<int64_t> hp(m + 1);
  CK(cudaMemcpyAsync(hp.data(), T.ptr, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  int64_t maxlen = 0;
  for (int64_t j = 0; j < m; ++j) maxlen = std::max(maxlen, hp[j + 1] - hp[j]);
  if (maxlen > kRankRow) {  // rows the rank sort skipped: block bitonic sort (shared memory or scratch)
    ++h->nlaunch;
    k_sort_rows<<<grid_for(m, 1, 148 * 32), 256, 0, h->stream>>>(T.ptr, m, T.ent, nullptr, 0);
  }
  if (maxlen > kRowSortCap) {
    int64_t np = 1;
    while (np < maxlen) np <<= 1;
    uint64_t* scr = h->alloc<uint64_t>(np);
    ++h->nlaunch; k_sort_rows<<<1, 256, 0, h->stream>>>(T.ptr, m, T.ent, scr, 1);
  }
  CKL("build_at");
  if (m0 == 0 && m1 == m) return T;
  // shard: keep rows [m0, m1) with local offsets
  DevCsr L;
  L.rows = m1 - m0;
  L.cols = A.rows;
  L.nnz = hp[m1] - hp[m0];
  L.ptr = h->alloc<int64_t>(L.rows + 1);
  std::vector<int64_t> lp(L.rows + 1);
  for (int64_t r = 0; r <= L.rows; ++r) lp[r] = hp[m0 + r] - hp[m0];
  CK(cudaMemcpy(L.ptr, lp.data(), sizeof(int64_t) * (L.rows + 1), cudaMemcpyHostToDevice));
  L.ent = T.ent + hp[m0];
  return L;
}

void init_u0(esnmf_t* h, const float* user_u0, bool on_dev) {
  Factor& f = h->U[0];
  const float* du = nullptr;
  if (user_u0) {
    if (on_dev) du = user_u0;
    else {
      float* tmp = h->alloc<float>(h->n * h->k);
      CK(cudaMemcpyAsync(tmp, user_u0, sizeof(float) * h->n * h->k, cudaMemcpyHostToDevice, h->stream));
      du = tmp;
    }
  }
  ++h->nlaunch; k_u0_dense<<<grid_for(h->n * h->kpad, 256, 148 * 32), 256, 0, h->stream>>>(h->n, h->k, h->kpad, h->seed, du,
                                                                               f.dense, h->flags + 2);
  if (h->init_nnz > 0 && !du) {
    // sparse U_0 (reading C18): mask the formula's entries, compact to COO, row view
    const double p = (double)h->init_nnz / (double)h->n;
    const uint64_t thr = p >= 1.0 ? ~0ULL : (uint64_t)(p * 0x1p53);
    h->nlaunch += 4;
    k_u0_mask<<<grid_for(h->n * h->k, 256, 148 * 32), 256, 0, h->stream>>>(h->n, h->k, h->kpad, h->seed, thr, f.dense);
    int64_t* cnt = h->side[ESNMF_SIDE_U].coltot;  // k scratch
    k_u0_compact<<<h->k, 1024, 0, h->stream>>>(h->n, h->k, h->kpad, f.dense, cnt, nullptr, f.row, f.val);
    k_sel_colptr<<<1, 256, 0, h->stream>>>(cnt, h->k, f.colptr);
    k_u0_compact<<<h->k, 1024, 0, h->stream>>>(h->n, h->k, h->kpad, f.dense, nullptr, f.colptr, f.row, f.val);
    CK(cudaMemsetAsync(f.dense, 0, sizeof(float) * h->n * h->kpad, h->stream));  // rebuilt for the active rows
    CKL("init_u0 sparse");
    f.has = true;
    factor_build_rows(h, f, h->n);
    h->ucur = 0;
    h->gramU_valid = false;
    return;
  }
  ++h->nlaunch; k_u0_coo<<<grid_for(h->n * h->k, 256, 148 * 32), 256, 0, h->stream>>>(h->n, h->k, h->kpad, f.dense, f.colptr,
                                                                          f.row, f.val, f.rowmap, f.active,
                                                                          f.n_active);
  CKL("init_u0");
  f.has = true;
  f.maxcol = h->n;
  h->ucur = 0;
  h->gramU_valid = false;
}

esnmf_status guard_status(const Fail& f) { return f.st; }

template <typename Fn>
esnmf_status guarded(Fn&& fn) {
  try {
    fn();
    return ESNMF_OK;
  } catch (const Fail& f) {
    return guard_status(f);
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return ESNMF_ENOMEM;
  } catch (...) {
    g_last_error = "unexpected exception";
    return ESNMF_ECUDA;
  }
}

void set_device(esnmf_t* h) { CK(cudaSetDevice(h->dev)); }

// the library's memory pool of a device (esnmf::alloc), created on first use
cudaMemPool_t device_pool(int dev) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (getenv("ESNMF_NO_POOL") || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CK(cudaMemPoolCreate(&pools[dev], &props));
    uint64_t never = ~0ull;
    CK(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &never));
  }
  return pools[dev];
}

}  // namespace

// =================================================================== C ABI

extern "C" {

const char* esnmf_version(void) { return "esnmf-b200 0.1 (sm_100a)"; }

const char* esnmf_strerror(esnmf_status s) {
  switch (s) {
    case ESNMF_OK: return "ok";
    case ESNMF_EINVAL: return "invalid argument";
    case ESNMF_ENOMEM: return "out of memory";
    case ESNMF_ECUDA: return "CUDA error";
    case ESNMF_ECOMM: return "collective failed";
    case ESNMF_ESINGULAR: return "singular Gram system";
    case ESNMF_EDEGENERATE: return "degenerate factor (||U|| = 0)";
    case ESNMF_ESTATE: return "call-order violation";
    case ESNMF_ETRUNC: return "buffer too small";
  }
  return "unknown status";
}

const char* esnmf_last_error(void) { return g_last_error.c_str(); }

esnmf_status esnmf_options_init(esnmf_options* o) {
  if (!o) return ESNMF_EINVAL;
  std::memset(o, 0, sizeof(*o));
  o->seed = 0;
  o->ridge_scale = 1e-10;
  o->device = -1;
  o->world = 1;
  o->rank = 0;
  o->head_terms = -1;
  o->t_u = ESNMF_T_SAME;
  o->t_v = ESNMF_T_SAME;
  o->enforce = ESNMF_ENFORCE_COLUMN;
  o->init_nnz = 0;
  o->seq_k2 = 0;
  o->seq_iters = 0;
  o->row_normalize = 0;
  o->keep_ls = 0;
  return ESNMF_OK;
}

esnmf_status esnmf_partition_rows(int64_t rows, const int64_t* row_ptr, int32_t world, int64_t* bounds) {
  if (rows < 0 || world < 1 || !bounds || (rows > 0 && !row_ptr)) {
    g_last_error = "esnmf_partition_rows: bad argument";
    return ESNMF_EINVAL;
  }
  // contiguous ranges balancing stored entries + rows (each row costs one item)
  const int64_t total = (rows > 0 ? row_ptr[rows] : 0) + rows;
  bounds[0] = 0;
  int64_t r = 0;
  for (int32_t p = 1; p < world; ++p) {
    const double target = (double)total * p / world;
    while (r < rows && (double)(row_ptr[r + 1] + r + 1) <= target) ++r;
    bounds[p] = r;
  }
  bounds[world] = rows;
  return ESNMF_OK;
}

// ESNMF_CREATE_TIMING=1: host wall time of each create stage (synchronised), to stderr
struct CreateTimer {
  bool on = getenv("ESNMF_CREATE_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(esnmf_t* h, const char* what) {
    if (!on) return;
    cudaStreamSynchronize(h->stream);
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "esnmf_create %-18s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

esnmf_status esnmf_create(esnmf_t** out, int64_t n, int64_t m, int32_t k, int64_t t, const int64_t* row_ptr,
                          const int32_t* col_idx, const float* val, const esnmf_options* opt) {
  CreateTimer ct;
  if (out) *out = nullptr;
  esnmf_options o;
  esnmf_options_init(&o);
  if (opt) o = *opt;
  if (!out || !row_ptr || !col_idx || !val) { g_last_error = "esnmf_create: NULL argument"; return ESNMF_EINVAL; }
  if (n < 1 || m < 1 || n >= (1LL << 31) || m >= (1LL << 31)) {
    g_last_error = "esnmf_create: need 1 <= n, m < 2^31 (got n=" + std::to_string(n) + ", m=" + std::to_string(m) + ")";
    return ESNMF_EINVAL;
  }
  if (k < 1 || k > ESNMF_MAX_K) { g_last_error = "esnmf_create: need 1 <= k <= 256"; return ESNMF_EINVAL; }
  if (t < 0 && t != ESNMF_T_UNLIMITED) { g_last_error = "esnmf_create: t must be >= 0 or ESNMF_T_UNLIMITED"; return ESNMF_EINVAL; }
  if (opt && ((opt->t_u < 0 && opt->t_u != ESNMF_T_UNLIMITED && opt->t_u != ESNMF_T_SAME) ||
              (opt->t_v < 0 && opt->t_v != ESNMF_T_UNLIMITED && opt->t_v != ESNMF_T_SAME))) {
    g_last_error = "esnmf_create: t_u / t_v must be >= 0, ESNMF_T_UNLIMITED or ESNMF_T_SAME";
    return ESNMF_EINVAL;
  }
  if (opt && opt->enforce != ESNMF_ENFORCE_COLUMN && opt->enforce != ESNMF_ENFORCE_MATRIX) {
    g_last_error = "esnmf_create: enforce must be ESNMF_ENFORCE_COLUMN or ESNMF_ENFORCE_MATRIX";
    return ESNMF_EINVAL;
  }
  if (opt && opt->enforce == ESNMF_ENFORCE_MATRIX && opt->world > 1) {
    g_last_error = "esnmf_create: whole-matrix enforcement is single-GPU only";
    return ESNMF_EINVAL;
  }
  if (o.seq_k2 != 0) {
    const char* why = nullptr;
    if (o.seq_k2 < 0 || k % o.seq_k2 != 0) why = "esnmf_create: seq_k2 must divide k";
    else if (o.seq_iters < 1) why = "esnmf_create: seq_iters must be >= 1 with seq_k2";
    else if (o.world > 1) why = "esnmf_create: sequential ALS is single-GPU only";
    else if (o.U0) why = "esnmf_create: sequential ALS draws its n x k2 U_0 itself (U0 must be NULL)";
    if (why) {
      g_last_error = why;
      return ESNMF_EINVAL;
    }
  }
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) { g_last_error = "esnmf_create: bad world/rank"; return ESNMF_EINVAL; }
  if (o.world > 1 && (!o.comm || !o.comm->allgather || !o.comm->allreduce_sum_f64)) {
    g_last_error = "esnmf_create: world > 1 needs comm callbacks";
    return ESNMF_EINVAL;
  }
  if (o.world > 64) { g_last_error = "esnmf_create: world must be <= 64"; return ESNMF_EINVAL; }
  if (!(o.ridge_scale >= 0) || !std::isfinite(o.ridge_scale)) { g_last_error = "esnmf_create: bad ridge_scale"; return ESNMF_EINVAL; }
  std::unique_ptr<esnmf> h(new esnmf());
  esnmf_status st = guarded([&] {
    if (o.device >= 0) h->dev = o.device;
    else CK(cudaGetDevice(&h->dev));
    set_device(h.get());
    if (o.stream) h->stream = (cudaStream_t)o.stream;
    else {
      CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      h->own_stream = true;
    }
    h->pool = device_pool(h->dev);
    {  // highest priority: its one-CTA solves must not queue behind the main stream's grids
      int least = 0, greatest = 0;
      CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      CK(cudaStreamCreateWithPriority(&h->aux, cudaStreamNonBlocking, greatest));
      CK(cudaStreamCreateWithPriority(&h->maux, cudaStreamNonBlocking, least));
    }
    for (cudaEvent_t* e : {&h->ev_ufork, &h->ev_ujoin, &h->ev_mfork, &h->ev_mjoin, &h->ev_vfork, &h->ev_vjoin,
                           &h->ev_gfork, &h->ev_gjoin, &h->ev_ugram})
      CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    h->n = n;
    h->m = m;
    h->keep_ls = o.keep_ls != 0;
    h->k = o.seq_k2 ? o.seq_k2 : k;  // sequential ALS: the pipeline works on one block
    h->kpad = (h->k + 3) / 4 * 4;
    const int32_t kb = h->k;  // columns of the pipeline (k, or k2 in sequential mode)
    if (o.seq_k2) {
      h->ktot = k;
      h->kpf = (k + 3) / 4 * 4;
      h->seq_k2 = o.seq_k2;
      h->seq_iters = o.seq_iters;
    }
    CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->dev));
    CK(cudaDeviceGetAttribute(&h->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
    h->t = t;
    h->tside[0] = o.t_v == ESNMF_T_SAME ? t : o.t_v;
    h->tside[1] = o.t_u == ESNMF_T_SAME ? t : o.t_u;
    h->whole = o.enforce == ESNMF_ENFORCE_MATRIX;
    h->init_nnz = o.init_nnz;
    if (h->whole && (int64_t)kb * (std::max(n, m) + 32) >= (1LL << 31))
      fail(ESNMF_EINVAL, "esnmf_create: whole-matrix enforcement needs k * rows < 2^31");
    h->wcolptr = h->alloc<int64_t>(2);
    if (const char* e = getenv("ESNMF_U_KMAX")) h->u_kmax = atof(e);
    h->rho = o.ridge_scale;
    h->seed = o.seed;
    h->world = o.world;
    h->rank = o.rank;
    if (o.comm) h->comm = *o.comm;
    h->sharded = h->world > 1 || (o.comm && getenv("ESNMF_FORCE_SHARDED"));
    const bool on_dev = o.inputs_on_device != 0;
    h->flags = h->alloc<int>(8);  // [0] singular [1] validation [2] U0 [3] U-side fp64 [4] V-side Z-gather fallback
    CK(cudaMemsetAsync(h->flags, 0, sizeof(int) * 8, h->stream));
    h->scal = h->alloc<double>(8);
    h->d_nrec = h->alloc<int64_t>(1);
    CK(cudaMemsetAsync(h->d_nrec, 0, sizeof(int64_t), h->stream));
    h->normA2_dev = h->alloc<double>(1);
    h->red_cap = 4LL * 2048 * 256 * 2;
    h->red = h->alloc<double>(h->red_cap);
    ct.mark(h.get(), "setup");
    // ---- row shards: terms nnz-balanced, documents equal ----
    std::vector<int64_t> hptr(n + 1);
    CK(cudaMemcpy(hptr.data(), row_ptr, sizeof(int64_t) * (n + 1),
                  on_dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    for (int64_t r = 0; r < n; ++r)
      if (hptr[r + 1] < hptr[r]) fail(ESNMF_EINVAL, "row_ptr is not non-decreasing at row " + std::to_string(r));
    std::vector<int64_t> ub(h->world + 1);
    esnmf_partition_rows(n, hptr.data(), h->world, ub.data());
    const int64_t n0 = ub[h->rank], n1 = ub[h->rank + 1];
    const int64_t m0 = m * h->rank / h->world, m1 = m * (h->rank + 1) / h->world;
    for (int p = 0; p < h->world; ++p) {
      h->u_rows_max = std::max(h->u_rows_max, ub[p + 1] - ub[p]);
      h->v_rows_max = std::max(h->v_rows_max, m * (p + 1) / h->world - m * p / h->world);
    }
    // ---- A (U side operator, this rank's term rows) ----
    std::vector<int64_t> aptr;
    Side& su = h->side[ESNMF_SIDE_U];
    su.row0 = n0;
    su.rows = n1 - n0;
    su.T = upload_csr(h.get(), n, m, row_ptr, col_idx, val, on_dev, n0, n1, &aptr);
    h->nnz = hptr[n];
    if (h->nnz < 1) fail(ESNMF_EINVAL, "esnmf_create: nnz must be >= 1");
    float* rowlen = nullptr;  // row normalisation: nnz of every term row of A
    if (o.row_normalize) {
      std::vector<float> rl(n);
      for (int64_t i = 0; i < n; ++i) rl[i] = (float)(hptr[i + 1] - hptr[i]);
      rowlen = h->alloc<float>(n);
      CK(cudaMemcpyAsync(rowlen, rl.data(), sizeof(float) * n, cudaMemcpyHostToDevice, h->stream));
      ++h->nlaunch;
      k_norm_rows<<<grid_for(su.rows, 8, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(su.T.ptr, su.T.ent, su.rows,
                                                                                        su.row0, rowlen);
      CK(cudaStreamSynchronize(h->stream));  // rl dies here
      CKL("norm_rows");
    }
    // ||A||_F^2 (shard partial, summed over ranks)
    {
      unsigned gb = grid_for(std::max<int64_t>(su.T.nnz, 1), 256, 1024);
      ++h->nlaunch; k_frob2<<<gb, 256, 0, h->stream>>>(su.T.ent, su.T.nnz, h->red);
      ++h->nlaunch; k_reduce_to<<<1, 256, 0, h->stream>>>(h->red, gb, h->normA2_dev);
      CKL("frob2");
      if (h->sharded && h->comm.allreduce_sum_f64(h->comm.ctx, h->normA2_dev, 1, h->stream) != 0)
        fail(ESNMF_ECOMM, "allreduce(||A||^2) failed");
    }
    ct.mark(h.get(), "upload A + norm");
    // ---- A^T (V side operator, this rank's document rows) ----
    Side& sv = h->side[ESNMF_SIDE_V];
    sv.row0 = m0;
    sv.rows = m1 - m0;
    bool at_normalized = false;
    if (o.at_row_ptr && o.at_col_idx && o.at_val) {
      sv.T = upload_csr(h.get(), m, n, o.at_row_ptr, o.at_col_idx, o.at_val, on_dev, m0, m1, nullptr);
    } else if (!h->sharded) {
      sv.T = build_at(h.get(), su.T, m, 0, m);  // from the (normalised) A
      at_normalized = true;
    } else {  // the transpose needs every term row: build it from the full A, keep our documents
      DevCsr full = upload_csr(h.get(), n, m, row_ptr, col_idx, val, on_dev, 0, n, nullptr);
      sv.T = build_at(h.get(), full, m, m0, m1);
    }
    if (rowlen && !at_normalized) {
      ++h->nlaunch;
      k_norm_cols<<<grid_for(std::max<int64_t>(sv.T.nnz, 1), 256, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(
          sv.T.ent, sv.T.nnz, rowlen);
      CKL("norm_cols");
    }
    if (!h->sharded && sv.T.nnz != h->nnz) fail(ESNMF_EINVAL, "esnmf_create: nnz(A^T) != nnz(A)");
    ct.mark(h.get(), "A^T");
    build_items(h.get(), su, aptr);
    side_alloc(h.get(), sv);
    ct.mark(h.get(), "items + V alloc");
    head_setup(h.get(), hptr, o.head_terms);
    ct.mark(h.get(), "head setup");
    side_alloc(h.get(), su);
    // ---- factors ----
    const int64_t capU = n * (int64_t)kb;
    const int64_t tv = h->tside[0];
    const int64_t capV = h->whole ? (tv < 0 ? m * (int64_t)kb : std::min(m * (int64_t)kb, std::max<int64_t>(tv, 1)))
                                  : (tv < 0 ? m : std::min(m, tv)) * (int64_t)kb;
    factor_alloc(h.get(), h->U[0], n, capU);
    factor_alloc(h.get(), h->U[1], n, capU);
    factor_alloc(h.get(), h->V, m, capV);
    {
      int G, CPL;
      tail_layout(h->kpad, G, CPL);

      // term-indexed Z rows, zero-padded to the gather layout (whole 16-byte
      // chunks per lane, no predicated loads)
      h->zs = 4 * G * CPL;
    }
    h->Z = h->alloc<float>(n * (int64_t)h->zs);
    CK(cudaMemsetAsync(h->Z, 0, sizeof(float) * n * (int64_t)h->zs, h->stream));
    h->zlist = h->alloc<int32_t>(n);
    if (narrow_v(h.get())) {
      const int kpz = h->k == 1 ? 1 : h->kpad;
      h->zc = h->alloc<float>(n * (int64_t)kpz);
      CK(cudaMemsetAsync(h->zc, 0, sizeof(float) * n * kpz, h->stream));
    }
    h->zcount = h->alloc<int64_t>(1);
    CK(cudaMemsetAsync(h->zcount, 0, sizeof(int64_t), h->stream));
    h->tbits = h->alloc<uint32_t>(ceil_div(n, 32));
    h->vbits = h->alloc<uint32_t>(ceil_div(m, 32));
    h->vmap = h->alloc<uint64_t>(m);
    h->vent = h->alloc<int2>(h->V.cap);
    h->vrptr = h->alloc<int64_t>(h->V.cap_rows + 1);
    h->vcur = h->alloc<int64_t>(h->V.cap_rows + 1);
    h->vscan = h->alloc<int64_t>(ceil_div(h->V.cap_rows + 1, kScanBlock) + 1);
    h->vmax = h->alloc<uint32_t>(1);
    h->rsum = h->alloc<double>(su.rows);
    ++h->nlaunch;
    k_rowsum<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(su.rows, (int64_t)h->num_sms * 8)), 256, 0,
               h->stream>>>(su.T.ptr, su.T.ent, su.rows, h->rsum);
    h->rsum_max = h->alloc<double>(1);
    ++h->nlaunch;
    k_max_to<<<1, 1024, 0, h->stream>>>(h->rsum, su.rows, h->rsum_max);
    if (!h->sharded) {
      h->W32 = h->alloc<float>((int64_t)kb * h->kpad);
      if (h->kpad <= 128 && !getenv("ESNMF_UTC_OFF")) {  // tensor-core (Y W), k_uside_tc.cuh
        h->utc_kn = (kb + 15) / 16 * 16;
        h->utc_kk = (h->kpad + 15) / 16 * 16;
        const int64_t wb = (int64_t)h->utc_kn * h->utc_kk * 4;
        h->wtc = h->alloc<uint8_t>(wb);
        CK(cudaMemsetAsync(h->wtc, 0, wb, h->stream));
        h->wtc_scale = h->alloc<float>(h->utc_kn);
        CK(cudaMemsetAsync(h->wtc_scale, 0, sizeof(float) * h->utc_kn, h->stream));
      }
      for (int b = 0; b < 2; ++b) {
        h->Yqb[b] = h->alloc<unsigned long long>(n * (int64_t)h->kpad);
        CK(cudaMemsetAsync(h->Yqb[b], 0, sizeof(unsigned long long) * n * h->kpad, h->stream));
      }
      h->Yq = h->Yqb[0];
    }
    CK(cudaMemsetAsync(h->vbits, 0, sizeof(uint32_t) * ceil_div(m, 32), h->stream));
    CK(cudaMemsetAsync(h->vmap, 0, sizeof(uint64_t) * m, h->stream));
    h->W = h->alloc<double>((int64_t)kb * kb);
    if (h->ktot) {  // converged columns (all blocks but the current one) and scratch
      const int eta = h->ktot / h->k;
      factor_alloc(h.get(), h->FU, n, h->U[0].cap * eta, h->ktot, h->kpf);
      factor_alloc(h.get(), h->FV, m, h->V.cap * eta, h->ktot, h->kpf);
      h->seqC = h->alloc<double>((int64_t)h->ktot * h->k);
      h->seqM = h->alloc<double>((int64_t)h->ktot * h->k);
      h->seqc = h->alloc<double>(4);
      CK(cudaMemsetAsync(h->seqc, 0, sizeof(double) * 4, h->stream));
    }
    h->gram_partial = h->alloc<double>((int64_t)std::max(kMaxGramSeg, kMaxGramSegDense) * kb * kb);
    if (kb > 128) h->sweep_scratch = h->alloc<double>((int64_t)kb * kb);  // blocked / packed sweep
    ct.mark(h.get(), "factors + buffers");
    init_u0(h.get(), o.U0, on_dev);
    ct.mark(h.get(), "U0");
    if (ct.on) fprintf(stderr, "esnmf_create cudaMalloc total   %8.2f ms (%zu buffers)\n", h->alloc_ms, h->allocs.size());
    CK(cudaStreamSynchronize(h->stream));
    int fl[4];
    CK(cudaMemcpy(fl, h->flags, sizeof(fl), cudaMemcpyDeviceToHost));
    if (fl[1]) {
      std::string why;
      if (fl[1] & 1) why += " row_ptr;";
      if (fl[1] & 2) why += " column index out of range;";
      if (fl[1] & 4) why += " column indices not strictly increasing within a row;";
      if (fl[1] & 8) why += " negative or non-finite value;";
      fail(ESNMF_EINVAL, "esnmf_create: malformed CSR:" + why);
    }
    if (fl[2]) fail(ESNMF_EINVAL, "esnmf_create: U0 must be finite and > 0");
    CK(cudaMemcpy(&h->normA2, h->normA2_dev, sizeof(double), cudaMemcpyDeviceToHost));
    if (!(h->normA2 > 0)) fail(ESNMF_EINVAL, "esnmf_create: ||A|| == 0");
  });
  if (st != ESNMF_OK) return st;
  *out = h.release();
  return ESNMF_OK;
}

esnmf_status esnmf_iterate(esnmf_t* h, int32_t iters) {
  if (!h || iters < 0) { g_last_error = "esnmf_iterate: bad argument"; return ESNMF_EINVAL; }
  return guarded([&] {
    set_device(h);
    ensure_records(h, h->nrec + iters);
    for (int32_t i = 0; i < iters; ++i) {
      if (graph_ok(h)) {
        graph_run(h);
      } else {
        iterate_one(h);
        ++h->steady;
      }
    }
    flush_metrics(h);  // the last iteration's record
    join_metrics(h);   // everything later on the caller's stream sees the records
  });
}

esnmf_status esnmf_half_step(esnmf_t* h, int32_t side) {
  if (!h || (side != ESNMF_SIDE_V && side != ESNMF_SIDE_U)) { g_last_error = "esnmf_half_step: bad argument"; return ESNMF_EINVAL; }
  return guarded([&] {
    set_device(h);
    graph_reset(h);
    h->force_ls = true;  // explicit half-steps always materialise the LS buffer
    half_step(h, side);
    h->force_ls = false;
    join_metrics(h);
    if (h->u_prefork) join_from_aux(h, h->ev_ujoin);  // callers may read G_V / W next
  });
}

static esnmf_status last_record(esnmf_t* h, esnmf_record* r) {
  return guarded([&] {
    set_device(h);
    if (h->nrec == 0) fail(ESNMF_ESTATE, "no completed iteration");
    sync_check(h);
    CK(cudaMemcpy(r, h->rec + h->nrec - 1, sizeof(esnmf_record), cudaMemcpyDeviceToHost));
  });
}

esnmf_status esnmf_residual(esnmf_t* h, double* R) {
  if (!h || !R) { g_last_error = "esnmf_residual: NULL argument"; return ESNMF_EINVAL; }
  esnmf_record r;
  esnmf_status st = last_record(h, &r);
  if (st != ESNMF_OK) return st;
  if (r.R < 0) { g_last_error = "residual undefined: ||U_i||_F == 0"; return ESNMF_EDEGENERATE; }
  *R = r.R;
  return ESNMF_OK;
}

esnmf_status esnmf_error(esnmf_t* h, double* E) {
  if (!h || !E) { g_last_error = "esnmf_error: NULL argument"; return ESNMF_EINVAL; }
  esnmf_record r;
  esnmf_status st = last_record(h, &r);
  if (st != ESNMF_OK) return st;
  *E = r.E;
  return ESNMF_OK;
}

esnmf_status esnmf_records(esnmf_t* h, int64_t cap, int64_t* count, esnmf_record* out) {
  if (!h || !count || cap < 0 || (cap > 0 && !out)) { g_last_error = "esnmf_records: bad argument"; return ESNMF_EINVAL; }
  esnmf_status st = guarded([&] {
    set_device(h);
    sync_check(h);
    *count = h->nrec;
    const int64_t nc = std::min(cap, h->nrec);
    if (nc > 0) CK(cudaMemcpy(out, h->rec, sizeof(esnmf_record) * nc, cudaMemcpyDeviceToHost));
  });
  if (st == ESNMF_OK && cap < h->nrec) { g_last_error = "esnmf_records: cap < count"; return ESNMF_ETRUNC; }
  return st;
}

// the factor's COO; in sequential mode the frozen columns [0, b0) (F1) first,
// then the block's k columns shifted to [b0, b0 + k)
static esnmf_status get_factor(esnmf_t* h, const Factor& f, int64_t cap, int64_t* nnz, int32_t* row, int32_t* col,
                               float* val, const Factor* F1 = nullptr) {
  if (!h || !nnz) { g_last_error = "get factor: NULL argument"; return ESNMF_EINVAL; }
  bool trunc = false;
  esnmf_status st = guarded([&] {
    set_device(h);
    sync_check(h);
    const int b0 = F1 ? h->seq_b * h->seq_k2 : 0;
    std::vector<int64_t> fp(b0 + 1, 0);
    if (b0 > 0) CK(cudaMemcpy(fp.data(), F1->colptr, sizeof(int64_t) * (b0 + 1), cudaMemcpyDeviceToHost));
    std::vector<int64_t> cp(h->k + 1, 0);
    if (f.has) CK(cudaMemcpy(cp.data(), f.colptr, sizeof(int64_t) * (h->k + 1), cudaMemcpyDeviceToHost));
    const int64_t nf = fp[b0], total = nf + cp[h->k];
    *nnz = total;
    if (cap < total || ((!row || !col || !val) && total > 0)) { trunc = true; return; }
    if (nf > 0) {
      CK(cudaMemcpy(row, F1->row, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(val, F1->val, sizeof(float) * nf, cudaMemcpyDeviceToHost));
      for (int c = 0; c < b0; ++c)
        for (int64_t e = fp[c]; e < fp[c + 1]; ++e) col[e] = c;
    }
    if (cp[h->k] > 0) {
      CK(cudaMemcpy(row + nf, f.row, sizeof(int32_t) * cp[h->k], cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(val + nf, f.val, sizeof(float) * cp[h->k], cudaMemcpyDeviceToHost));
      for (int c = 0; c < h->k; ++c)
        for (int64_t e = cp[c]; e < cp[c + 1]; ++e) col[nf + e] = b0 + c;
    }
  });
  if (st == ESNMF_OK && trunc) { g_last_error = "factor buffer too small"; return ESNMF_ETRUNC; }
  return st;
}

esnmf_status esnmf_get_U(esnmf_t* h, int64_t cap, int64_t* nnz, int32_t* row, int32_t* col, float* val) {
  if (!h) { g_last_error = "NULL handle"; return ESNMF_EINVAL; }
  return get_factor(h, h->U[h->ucur], cap, nnz, row, col, val, h->ktot ? &h->FU : nullptr);
}

esnmf_status esnmf_get_V(esnmf_t* h, int64_t cap, int64_t* nnz, int32_t* row, int32_t* col, float* val) {
  if (!h) { g_last_error = "NULL handle"; return ESNMF_EINVAL; }
  return get_factor(h, h->V, cap, nnz, row, col, val, h->ktot ? &h->FV : nullptr);
}

esnmf_status esnmf_set_factor(esnmf_t* h, int32_t side, int64_t nnz, const int32_t* row, const int32_t* col,
                              const float* val) {
  if (!h || (side != ESNMF_SIDE_V && side != ESNMF_SIDE_U) || nnz < 0 || (nnz > 0 && (!row || !col || !val))) {
    g_last_error = "esnmf_set_factor: bad argument";
    return ESNMF_EINVAL;
  }
  Factor& f = side == ESNMF_SIDE_U ? h->U[h->ucur] : h->V;
  const int64_t rows = side == ESNMF_SIDE_U ? h->n : h->m;
  // validate canonical order on the host
  std::vector<int64_t> cp(h->k + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) {
    if (col[e] < 0 || col[e] >= h->k || row[e] < 0 || row[e] >= rows || !(val[e] > 0.f) || !std::isfinite(val[e])) {
      g_last_error = "esnmf_set_factor: entry " + std::to_string(e) + " out of range or not > 0";
      return ESNMF_EINVAL;
    }
    if (e > 0 && (col[e] < col[e - 1] || (col[e] == col[e - 1] && row[e] <= row[e - 1]))) {
      g_last_error = "esnmf_set_factor: entries not in canonical (column, row) order";
      return ESNMF_EINVAL;
    }
    cp[col[e] + 1]++;
  }
  for (int c = 0; c < h->k; ++c) cp[c + 1] += cp[c];
  int64_t maxcol = 0;
  for (int c = 0; c < h->k; ++c) maxcol = std::max(maxcol, cp[c + 1] - cp[c]);
  if (nnz > f.cap) { g_last_error = "esnmf_set_factor: more entries than the factor capacity"; return ESNMF_EINVAL; }
  return guarded([&] {
    set_device(h);
    graph_reset(h);
    CK(cudaStreamSynchronize(h->aux));
    CK(cudaStreamSynchronize(h->maux));
    if (side == ESNMF_SIDE_V) vrows_clear(h);
    factor_clear(h, f);
    CK(cudaMemcpyAsync(f.colptr, cp.data(), sizeof(int64_t) * (h->k + 1), cudaMemcpyHostToDevice, h->stream));
    if (nnz > 0) {
      CK(cudaMemcpyAsync(f.row, row, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, h->stream));
      CK(cudaMemcpyAsync(f.val, val, sizeof(float) * nnz, cudaMemcpyHostToDevice, h->stream));
    }
    factor_build_rows(h, f, std::max<int64_t>(maxcol, 1));
    if (side == ESNMF_SIDE_V) {
      vrows_build(h);
      h->u_prefork = false;  // a pre-started U-side Gram belongs to the old V
    }
    if (side == ESNMF_SIDE_U) h->gramU_valid = false;
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaStreamSynchronize(h->aux));
    CK(cudaStreamSynchronize(h->maux));
  });
}

esnmf_status esnmf_truncate(esnmf_t* h, int32_t side, int64_t t, int32_t enforce) {
  if (!h || (side != ESNMF_SIDE_V && side != ESNMF_SIDE_U) || t < 0 ||
      (enforce != ESNMF_ENFORCE_COLUMN && enforce != ESNMF_ENFORCE_MATRIX)) {
    g_last_error = "esnmf_truncate: bad argument";
    return ESNMF_EINVAL;
  }
  if (h->sharded) { g_last_error = "esnmf_truncate: single GPU only"; return ESNMF_EINVAL; }
  return guarded([&] {
    set_device(h);
    graph_reset(h);
    CK(cudaStreamSynchronize(h->aux));
    CK(cudaStreamSynchronize(h->maux));
    Factor& f = side == ESNMF_SIDE_U ? h->U[h->ucur] : h->V;
    if (!f.has) fail(ESNMF_ESTATE, "esnmf_truncate: factor not set");
    Side& sd = h->side[side];  // its LS buffer is the scratch
    const int k = h->k;
    CK(cudaMemsetAsync(sd.X, 0, sizeof(float) * k * sd.ldx, h->stream));
    ++h->nlaunch;
    k_coo_to_colmajor<<<dim3(col_grid_x(f.maxcol), k), 256, 0, h->stream>>>(f.colptr, f.row, f.val, sd.X, sd.ldx);
    if (side == ESNMF_SIDE_V) vrows_clear(h);
    factor_clear(h, f);
    if (enforce == ESNMF_ENFORCE_COLUMN) {
      select_core(h, sd, sd.X, sd.ldx, sd.rows, k, 0, t, false, f.colptr, f.row, f.val, nullptr);
    } else {
      select_core(h, sd, sd.X, (int64_t)k * sd.ldx, (int64_t)k * sd.ldx, 1, 0, t, false, h->wcolptr, f.row, f.val,
                  nullptr);
      h->nlaunch += 2;
      k_whole_colptr<<<1, 256, 0, h->stream>>>(f.row, h->wcolptr, sd.ldx, k, f.colptr);
      k_whole_rows<<<grid_for(f.cap, 256, (int64_t)h->num_sms * 8), 256, 0, h->stream>>>(f.row, h->wcolptr,
                                                                                        sd.ldx);
    }
    factor_build_rows(h, f, std::min<int64_t>(f.rows, std::max<int64_t>(t, 1)));
    if (side == ESNMF_SIDE_V) vrows_build(h);
    if (side == ESNMF_SIDE_U) h->gramU_valid = false;
    h->u_prefork = false;
    sd.ls_valid = false;  // the scratch overwrote the LS rows
    CK(cudaStreamSynchronize(h->stream));
  });
}

esnmf_status esnmf_get_ls(esnmf_t* h, int32_t side, int64_t* row0, int64_t* rows, float* out) {
  if (!h || (side != ESNMF_SIDE_V && side != ESNMF_SIDE_U)) { g_last_error = "esnmf_get_ls: bad argument"; return ESNMF_EINVAL; }
  Side& sd = h->side[side];
  if (row0) *row0 = sd.row0;
  if (rows) *rows = sd.rows;
  if (!out) return ESNMF_OK;
  return guarded([&] {
    set_device(h);
    if (!sd.ls_valid) fail(ESNMF_ESTATE, "no half-step of this side has run");
    if (!sd.ls_stored)
      fail(ESNMF_ESTATE, "the V side's LS buffer was not written by esnmf_iterate (esnmf_options.keep_ls = 1, "
                         "or esnmf_half_step)");
    sync_check(h);
    std::vector<float> buf((size_t)h->k * sd.ldx);
    CK(cudaMemcpy(buf.data(), sd.X, sizeof(float) * buf.size(), cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < sd.rows; ++r)
      for (int c = 0; c < h->k; ++c) out[r * h->k + c] = buf[(size_t)c * sd.ldx + r];
  });
}

esnmf_status esnmf_get_gram(esnmf_t* h, int32_t side, double* G, double* eps) {
  if (!h || (side != ESNMF_SIDE_V && side != ESNMF_SIDE_U) || !G) { g_last_error = "esnmf_get_gram: bad argument"; return ESNMF_EINVAL; }
  return guarded([&] {
    set_device(h);
    // Gram of the factor this side reads next (side V: U^T U, side U: V^T V),
    // recomputed by the same kernels into a scratch buffer.
    const Factor& f = side == ESNMF_SIDE_V ? h->U[h->ucur] : h->V;
    if (!f.has) fail(ESNMF_ESTATE, "factor not set");
    double* Gd = h->W;  // W is rebuilt by every half-step: free between calls
    gram(h, f, Gd);
    sync_check(h);
    CK(cudaMemcpy(G, Gd, sizeof(double) * h->k * h->k, cudaMemcpyDeviceToHost));
    if (eps) {
      double tr = 0;
      for (int a = 0; a < h->k; ++a) tr += G[a * h->k + a];
      *eps = h->rho * (tr / h->k + 1.0);
    }
  });
}

esnmf_status esnmf_nccl_unique_id(void* id) {
  if (!id) { g_last_error = "esnmf_nccl_unique_id: NULL"; return ESNMF_EINVAL; }
  const NcclApi& a = nccl_api();
  if (!a.error.empty()) { g_last_error = a.error; return ESNMF_ECOMM; }
  ncclUniqueId u;
  const ncclResult_t r = a.getUniqueId(&u);
  if (r != ncclSuccess) { g_last_error = std::string("ncclGetUniqueId: ") + a.getErrorString(r); return ESNMF_ECOMM; }
  static_assert(sizeof(ncclUniqueId) == ESNMF_NCCL_ID_BYTES, "NCCL unique id size");
  std::memcpy(id, &u, sizeof(u));
  return ESNMF_OK;
}

esnmf_status esnmf_nccl_comm_create(int32_t world, int32_t rank, const void* id, int32_t device, esnmf_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) {
    g_last_error = "esnmf_nccl_comm_create: bad argument";
    return ESNMF_EINVAL;
  }
  *out = nullptr;
  const NcclApi& a = nccl_api();
  if (!a.error.empty()) { g_last_error = a.error; return ESNMF_ECOMM; }
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) { g_last_error = "cudaSetDevice failed"; return ESNMF_ECUDA; }
  auto* ctx = new NcclCtx();
  ctx->world = world;
  ctx->rank = rank;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  const ncclResult_t r = a.commInitRank(&ctx->comm, world, u, rank);
  if (r != ncclSuccess) {
    g_last_error = std::string("ncclCommInitRank: ") + a.getErrorString(r);
    delete ctx;
    return ESNMF_ECOMM;
  }
  auto* c = new esnmf_comm();
  c->ctx = ctx;
  c->allgather = nccl_allgather_cb;
  c->allreduce_sum_f64 = nccl_allreduce_cb;
  *out = c;
  return ESNMF_OK;
}

void esnmf_nccl_comm_destroy(esnmf_comm* c) {
  if (!c) return;
  if (builtin_nccl(*c)) {
    auto* ctx = static_cast<NcclCtx*>(c->ctx);
    if (ctx->comm) nccl_api().commDestroy(ctx->comm);
    delete ctx;
  }
  delete c;
}

esnmf_status esnmf_cost_model(esnmf_t* h, esnmf_cost* out) {
  if (!h || !out) { g_last_error = "esnmf_cost_model: NULL argument"; return ESNMF_EINVAL; }
  return guarded([&] {
    set_device(h);
    if (!h->V.has) fail(ESNMF_ESTATE, "no V side has run");
    std::memset(out, 0, sizeof(*out));
    Side& sv = h->side[ESNMF_SIDE_V];
    out->head_terms = h->head_h;
    out->paper_order_tail = h->ptail ? 1 : 0;
    double* d = h->red;  // scratch
    CK(cudaMemsetAsync(d, 0, sizeof(double), h->stream));
    ++h->nlaunch;
    k_u_cost<<<grid_for(h->V.cap, 256, (int64_t)h->num_sms * 4), 256, 0, h->stream>>>(
        h->V.colptr, h->V.row, h->k, sv.row0, sv.rows, sv.T.ptr, d);
    CKL("u_cost");
    sync_check(h);
    CK(cudaMemcpy(&out->u_products, d, sizeof(double), cudaMemcpyDeviceToHost));
    if (h->head_ntiles > 0) {
      const double tiles = (double)h->head_ntiles;
      out->v_head_mma_flops = tiles * 128.0 * (double)h->head_h * h->kn * 2.0 * 3.0;
    }
    if (h->ptail) {
      double c[8];
      int fl[8];
      CK(cudaMemcpy(c, h->vcost, sizeof(c), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(fl, h->flags, sizeof(fl), cudaMemcpyDeviceToHost));
      out->v_tail_products = c[0];
      out->v_tail_gather_fma = c[1];
      out->v_tail_active = c[2];
      out->v_head_products = c[3];
      out->v_tail_gather = fl[4];
      out->v_gather_by_cost = fl[5];
      if (!fl[4]) out->v_yw_mma_flops = (double)h->head_ntiles * 128.0 * h->kn * h->kn * 2.0 * 3.0;
    } else {
      out->v_tail_gather = 1;
    }
  });
}

esnmf_status esnmf_profile(esnmf_t* h, int32_t enable) {
  if (!h) { g_last_error = "esnmf_profile: NULL handle"; return ESNMF_EINVAL; }
  return guarded([&] {
    set_device(h);
    CK(cudaStreamSynchronize(h->stream));
    prof_collect(h);
    for (int i = 0; i < kNumPhases; ++i) { h->prof_ms[i] = 0; h->prof_calls[i] = 0; }
    h->prof_on = enable != 0;
  });
}

esnmf_status esnmf_phase_times(esnmf_t* h, int64_t cap, int64_t* count, esnmf_phase* out) {
  if (!h || !count || cap < 0 || (cap > 0 && !out)) { g_last_error = "esnmf_phase_times: bad argument"; return ESNMF_EINVAL; }
  esnmf_status st = guarded([&] {
    set_device(h);
    CK(cudaStreamSynchronize(h->stream));
    prof_collect(h);
    *count = kNumPhases;
    for (int i = 0; i < kNumPhases && i < cap; ++i) {
      std::memset(out[i].name, 0, sizeof(out[i].name));
      std::strncpy(out[i].name, kPhaseNames[i], sizeof(out[i].name) - 1);
      out[i].calls = h->prof_calls[i];
      out[i].ms = h->prof_ms[i];
    }
  });
  if (st == ESNMF_OK && cap < kNumPhases) { g_last_error = "esnmf_phase_times: cap < count"; return ESNMF_ETRUNC; }
  return st;
}

esnmf_status esnmf_topic_accuracy(esnmf_t* h, const int32_t* labels, int32_t n_journals, double* acc) {
  if (!h || !labels || !acc || n_journals < 1) { g_last_error = "esnmf_topic_accuracy: bad argument"; return ESNMF_EINVAL; }
  for (int64_t j = 0; j < h->m; ++j)
    if (labels[j] < 0 || labels[j] >= n_journals) {
      g_last_error = "esnmf_topic_accuracy: label " + std::to_string(j) + " out of [0, n_journals)";
      return ESNMF_EINVAL;
    }
  return guarded([&] {
    set_device(h);
    join_metrics(h);
    if (!h->V.has) fail(ESNMF_ESTATE, "V is not set");
    const int kt = h->ktot ? h->ktot : h->k;
    struct Tmp {  // per-call scratch, freed on every exit
      void* p = nullptr;
      ~Tmp() { if (p) cudaFree(p); }
    } tl, tc;
    CK(cudaMalloc(&tl.p, sizeof(int32_t) * h->m));
    CK(cudaMalloc(&tc.p, sizeof(double) * ((int64_t)kt * n_journals + kt)));
    int32_t* dl = static_cast<int32_t*>(tl.p);
    double* cnt = static_cast<double*>(tc.p);
    double* dacc = cnt + (int64_t)kt * n_journals;
    CK(cudaMemcpyAsync(dl, labels, sizeof(int32_t) * h->m, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemsetAsync(cnt, 0, sizeof(double) * kt * n_journals, h->stream));
    const int b0 = h->ktot ? h->seq_b * h->seq_k2 : 0;
    if (b0 > 0) {
      ++h->nlaunch;
      k_acc_count<<<dim3(col_grid_x(h->FV.maxcol), b0), 256, 0, h->stream>>>(h->FV.colptr, h->FV.row, dl,
                                                                             n_journals, 0, cnt);
    }
    h->nlaunch += 2;
    k_acc_count<<<dim3(col_grid_x(h->V.maxcol), h->k), 256, 0, h->stream>>>(h->V.colptr, h->V.row, dl, n_journals,
                                                                            b0, cnt);
    k_acc_final<<<1, 256, 0, h->stream>>>(cnt, kt, n_journals, dacc);
    CK(cudaMemcpyAsync(acc, dacc, sizeof(double) * kt, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    CKL("topic_accuracy");
  });
}

esnmf_status esnmf_get_info(esnmf_t* h, esnmf_info* info) {
  if (!h || !info) { g_last_error = "esnmf_get_info: NULL argument"; return ESNMF_EINVAL; }
  info->n = h->n;
  info->m = h->m;
  info->nnz = h->nnz;
  info->k = h->ktot ? h->ktot : h->k;
  info->ls_cols = h->k;
  info->seq_block = h->seq_b;
  info->t = h->t;
  info->world = h->world;
  info->rank = h->rank;
  info->v_row0 = h->side[0].row0;
  info->v_rows = h->side[0].rows;
  info->u_row0 = h->side[1].row0;
  info->u_rows = h->side[1].rows;
  info->iterations = h->nrec;
  info->device_bytes = h->bytes;
  info->normA2 = h->normA2;
  info->launches = h->nlaunch;
  info->head_terms = h->head_h;
  info->head_dense = h->head_nd;
  return ESNMF_OK;
}

void esnmf_destroy(esnmf_t* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  delete h;
}

}  // extern "C"
