// extern "C" boundary (include/skewgcn_b200.h): graph store, plan arenas, orchestration.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <thread>

#include <unistd.h>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/skewgcn_b200.h"
#include "gcn.cuh"
#include "prof.h"
#include "sampler.cuh"
#include "skg_internal.h"

namespace skg {
// per-kernel event timing (bench.py roofline): target "*" brackets every launch, else the
// launches whose name equals the target; pairs are kept per launch name
static std::string g_prof_target;
struct ProfPair {
  std::string name;
  cudaEvent_t a, b;
};
static std::vector<ProfPair> g_prof_pairs;
static cudaEvent_t g_prof_open = nullptr;
static std::string g_prof_open_name;
bool prof_match(const char* name) {
  if (g_prof_target.empty()) return false;
  if (g_prof_target == "*" || g_prof_target == name) {
    g_prof_open_name = name;
    return true;
  }
  return false;
}

// CUDA graphs of fixed launch sequences (the training step, the LADIES sampler): the
// per-call host cost of ~50-90 launches was the throughput limit.  A sequence is captured
// once per key (everything its launches bake in) on a private stream and replayed with one
// cudaGraphLaunch; per-call inputs live in device memory written before the replay.
struct GraphEntry {
  cudaGraphExec_t exec;
  unsigned long long launches;  // kernels per replay (for the launch counter)
};
struct GraphCache {
  std::unordered_map<std::string, GraphEntry> map;
  std::unordered_map<std::string, int> seen;  // keys run eagerly once (captured on reuse)
  cudaStream_t cap = nullptr;
  ~GraphCache() { clear(); }
  void clear() {
    for (auto& kv : map) cudaGraphExecDestroy(kv.second.exec);
    map.clear();
    seen.clear();
  }
};

// capture-only mode (skg_set_capture_only): graph_run records and instantiates a launch
// sequence without replaying it, so a benchmark can build every graph it will replay
// before its warm-up (no capture inside a timed region, warm-up exactly as requested)
static int g_capture_only = 0;

bool graphs_on() {
  static const int on = getenv("SKG_GCN_GRAPH") ? atoi(getenv("SKG_GCN_GRAPH")) : 1;
  return on != 0 && g_prof_target.empty();  // per-kernel profiling needs eager launches
}

// repeat: the caller reuses its keys (Trainer steps, sampler calls): capture at once.
// Otherwise a key's first use runs eagerly and its second use captures, so one-off calls
// (loss_and_backward on freshly allocated weights) never pay a capture.
template <typename Fn>
int graph_run(GraphCache& gc, const std::string& key, cudaStream_t st, bool repeat, Fn&& launch) {
  auto it = gc.map.find(key);
  if (it == gc.map.end()) {
    if (!repeat && !g_capture_only) {
      if (gc.seen.size() > 4096) gc.seen.clear();
      if (gc.seen[key]++ == 0) return launch(st);
    }
    if (!gc.cap && cudaStreamCreateWithFlags(&gc.cap, cudaStreamNonBlocking) != cudaSuccess) {
      set_error("graph capture stream");
      return SKG_ERR_CUDA;
    }
    const unsigned long long l0 = g_kernel_launches;
    if (cudaStreamBeginCapture(gc.cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      set_error("graph capture begin");
      return SKG_ERR_CUDA;
    }
    int rc = launch(gc.cap);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(gc.cap, &graph);
    const unsigned long long nl = g_kernel_launches - l0;
    g_kernel_launches = l0;  // capturing launched nothing
    if (rc || ce != cudaSuccess || !graph) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      if (rc) return rc;
      set_error(std::string("graph capture: ") + cudaGetErrorString(ce));
      return SKG_ERR_CUDA;
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      set_error(std::string("graph instantiate: ") + cudaGetErrorString(ie));
      return SKG_ERR_CUDA;
    }
    if (gc.map.size() >= 256) {  // bound the cache
      for (auto& kv : gc.map) cudaGraphExecDestroy(kv.second.exec);
      gc.map.clear();
    }
    it = gc.map.emplace(key, GraphEntry{exec, nl}).first;
  }
  if (g_capture_only) return SKG_OK;
  if (cudaGraphLaunch(it->second.exec, st) != cudaSuccess) {
    set_error(std::string("graph launch: ") + cudaGetErrorString(cudaGetLastError()));
    return SKG_ERR_CUDA;
  }
  g_kernel_launches += it->second.launches;
  return SKG_OK;
}

template <typename T>
void key_put(std::string& k, const T& v) {
  k.append(reinterpret_cast<const char*>(&v), sizeof(T));
}
void prof_record(cudaStream_t st, bool before) {
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  if (before) g_prof_open = e;
  else g_prof_pairs.push_back({g_prof_open_name, g_prof_open, e});
}
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }
}  // namespace skg

using namespace skg;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      set_error(std::string(#x) + ": " + cudaGetErrorString(e_));                    \
      return SKG_ERR_CUDA;                                                           \
    }                                                                                \
  } while (0)
#define ARG(cond, msg)       \
  do {                       \
    if (!(cond)) {           \
      set_error(msg);        \
      return SKG_ERR_ARG;    \
    }                        \
  } while (0)


// ------------------------------------------------------------------ structures
struct skg_ctx {
  int device = 0;
  int64_t n = 0, nnz = 0;
  int32_t n_workers = 1;
  int64_t* d_off = nullptr;
  int32_t* d_col = nullptr;
  double* d_w = nullptr;
  int32_t* d_owner = nullptr;
  int64_t* d_toff = nullptr;
  int32_t* d_trow = nullptr;
  double* d_tw = nullptr;
  bool symmetric = true;
  bool normalized = false;
  double* d_degd = nullptr;
  // fused range expand tables (normalised graphs), one per range size, built on first use
  bool fr_ok = false;
  std::unordered_map<int, int32_t*> rstarts;
  std::vector<int64_t> deg_desc_prefix;  // prefix sums of degrees sorted descending
  void* d_x = nullptr;
  int64_t F = 0, ldx = 0, x_rows = 0;
  int xbits = 0;  // 1: d_x holds bit-packed multi-hot rows (ldx 32-bit words per row)
  int dtype = DT_F32;
  int32_t* d_labels = nullptr;
  // multi-label targets (multi-hot, y_words 64-bit words per node) for the BCE loss
  uint64_t* d_ymulti = nullptr;
  int32_t y_words = 0, y_classes = 0;
  int n_ranks = 1;
  uint64_t* d_shards = nullptr;
  int32_t* d_node_rank = nullptr;
  int32_t* d_node_row = nullptr;
  std::vector<void*> shards_owned;
  uint64_t gen = 0;  // bumped by every setter: captured GCN graphs bake these pointers in
  GraphDev gdev() const {
    GraphDev g;
    g.n = n;
    g.nnz = nnz;
    g.off = d_off;
    g.col = d_col;
    g.w = d_w;
    g.owner = d_owner;
    g.t_off = symmetric ? d_off : d_toff;
    g.t_row = symmetric ? d_col : d_trow;
    g.t_w = symmetric ? d_w : d_tw;
    g.n_words = (int32_t)((n + 31) / 32);
    g.normalized = normalized ? 1 : 0;
    g.degd = d_degd;
    g.rstart = nullptr;  // per plan set (skg_plans::rstart)
    g.n_fr = 0;
    g.fr_size = 0;
    return g;
  }
  FeatStore fstore() const {
    FeatStore fs;
    fs.shards = reinterpret_cast<const void* const*>(d_shards);
    fs.node_rank = d_node_rank;
    fs.node_row = d_node_row;
    fs.ld = ldx;
    fs.dim = F;
    fs.bits = xbits;
    fs.pad_ = 0;
    return fs;
  }
  int64_t edge_bound(int64_t rows) const {  // max sum of `rows` distinct row degrees
    if (rows <= 0) return 0;
    rows = std::min<int64_t>(rows, (int64_t)deg_desc_prefix.size() - 1);
    return deg_desc_prefix[rows];
  }
};

struct skg_plans {
  skg_ctx* ctx = nullptr;
  int kind = KIND_LADIES, n_slots = 0, L = 0;
  int64_t budget = 0, max_batch = 0;
  int cap_rows = 0, cap_cand = 0, cap_batch = 0;
  int64_t cap_pairs = 0;
  int n_fr = 0;  // fused range expand: ranges per plan (0: the older expand kernels)
  int fr_size = 0;  // nodes per range
  const int32_t* rstart = nullptr;  // the context's table for fr_size
  std::vector<PlanDev> h;
  PlanDev* d_plans = nullptr;
  char* arena = nullptr;
  size_t scal_bytes = 0;
  char* d_scal = nullptr;  // per-slot scalars zeroed before each sampling call
  int32_t* d_batch = nullptr;
  // SAINT candidates
  int32_t* d_train = nullptr;
  double* d_train_norm = nullptr;
  uint32_t* d_train_bitmap = nullptr;
  int64_t n_train = 0;
  bool have_train_norm = false;
  std::vector<int32_t*> d_local;
  std::vector<double*> d_local_norm;
  std::vector<int64_t> n_local;
  std::vector<bool> local_norm_ready;
  GraphCache graphs;  // LADIES launch sequences per (plans, rows cap, context generation)
  // sticky error bits: every consumed plan's err word is OR-ed in by k_ledger_add (after
  // its training step), so an error survives the arena's reuse by the next sampling call
  int32_t* d_sticky = nullptr;
  // pinned staging of each sampling call's uploads (descriptors, batch ids); up_ev marks
  // the last upload consumed by its stream before the host rewrites the staging
  PlanDev* h_pin = nullptr;
  int32_t* hb_pin = nullptr;
  // explicit-uniform streams (SKG_RNG_EXPLICIT): n_slots x (L * budget) doubles, staged in
  // pinned memory and uploaded with the descriptors
  double* hu_pin = nullptr;
  double* d_unif = nullptr;
  size_t unif_staged = 0;
  cudaEvent_t up_ev = nullptr;
  bool up_armed = false;
};

// wait until the previous upload from the pinned staging has been consumed
int staging_ready(skg_plans* ps) {
  if (!ps->h_pin) {
    CK(cudaHostAlloc(reinterpret_cast<void**>(&ps->h_pin), sizeof(PlanDev) * std::max(ps->n_slots, 1),
                     cudaHostAllocDefault));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&ps->hb_pin),
                     sizeof(int32_t) * std::max<size_t>((size_t)ps->n_slots * ps->cap_batch, 1),
                     cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&ps->up_ev, cudaEventDisableTiming));
  }
  if (ps->up_armed) CK(cudaEventSynchronize(ps->up_ev));
  ps->up_armed = false;
  return SKG_OK;
}

// descriptors of the first n slots (and nb batch ids, when given) -> device, async
int upload_plans(skg_plans* ps, int n, size_t nb, cudaStream_t st) {
  std::memcpy(ps->h_pin, ps->h.data(), sizeof(PlanDev) * n);
  CK(cudaMemcpyAsync(ps->d_plans, ps->h_pin, sizeof(PlanDev) * n, cudaMemcpyHostToDevice, st));
  if (nb) CK(cudaMemcpyAsync(ps->d_batch, ps->hb_pin, sizeof(int32_t) * nb, cudaMemcpyHostToDevice, st));
  if (ps->unif_staged) {
    CK(cudaMemcpyAsync(ps->d_unif, ps->hu_pin, sizeof(double) * ps->unif_staged, cudaMemcpyHostToDevice, st));
    ps->unif_staged = 0;
  }
  CK(cudaEventRecord(ps->up_ev, st));
  ps->up_armed = true;
  return SKG_OK;
}

// slot i's uniform stream: `rngs[i]`, or the PCG64 words pcg[4i..4i+3] (older entry points).
// Explicit uniforms are staged for upload_plans (after staging_ready, so the pinned buffer
// is free); their count is capped to the n_layers * budget draws a plan can make.
int set_rng(skg_plans* ps, PlanDev& P, int i, const skg_rng* rngs, const uint64_t* pcg) {
  P.rng_kind = RNG_PCG64;
  P.rng_pos = 4;
  P.uniforms = nullptr;
  P.n_uniforms = 0;
  if (!rngs) {
    for (int q = 0; q < 4; ++q) P.rng[q] = pcg[4 * i + q];
    return SKG_OK;
  }
  const skg_rng& r = rngs[i];
  if (r.kind == SKG_RNG_PCG64) {
    for (int q = 0; q < 4; ++q) P.rng[q] = r.w[q];
  } else if (r.kind == SKG_RNG_PHILOX) {
    if (r.buffer_pos < 0 || r.buffer_pos > 4) {
      set_error("Philox buffer_pos out of range");
      return SKG_ERR_ARG;
    }
    P.rng_kind = RNG_PHILOX;
    P.rng_pos = r.buffer_pos;
    for (int q = 0; q < 10; ++q) P.phx[q] = r.w[q];
  } else if (r.kind == SKG_RNG_EXPLICIT) {
    if (!r.uniforms || r.n_uniforms < 0) {
      set_error("explicit uniform stream without uniforms");
      return SKG_ERR_ARG;
    }
    const size_t per = (size_t)ps->L * (size_t)ps->budget;
    if (!ps->hu_pin) {
      CK(cudaHostAlloc(reinterpret_cast<void**>(&ps->hu_pin), sizeof(double) * per * ps->n_slots,
                       cudaHostAllocDefault));
      CK(cudaMalloc(&ps->d_unif, sizeof(double) * per * ps->n_slots));
    }
    const size_t cnt = std::min<size_t>((size_t)r.n_uniforms, per);
    std::memcpy(ps->hu_pin + (size_t)i * per, r.uniforms, sizeof(double) * cnt);
    ps->unif_staged = std::max(ps->unif_staged, (size_t)i * per + cnt);
    P.rng_kind = RNG_EXPLICIT;
    P.uniforms = ps->d_unif + (size_t)i * per;
    P.n_uniforms = (int64_t)cnt;
  } else {
    set_error("unknown rng kind");
    return SKG_ERR_ARG;
  }
  return SKG_OK;
}

// the LADIES launch sequence for the first n slots (descriptors already on the device)
int run_ladies(skg_plans* ps, int n, int max_upper, cudaStream_t st) {
  skg_ctx* c = ps->ctx;
  auto launch = [&](cudaStream_t s) {
    GraphDev g = c->gdev();
    g.rstart = ps->rstart;
    g.n_fr = ps->n_fr;
    g.fr_size = ps->fr_size;
    return launch_ladies(g, ps->d_plans, n, ps->L, max_upper, ps->cap_cand, ps->cap_pairs,
                         (int)ps->budget, ps->n_fr, s);
  };
  if (!graphs_on()) return launch(st);
  std::string key;
  key_put(key, n);
  key_put(key, max_upper);
  key_put(key, c->gen);
  return graph_run(ps->graphs, key, st, true, launch);
}

struct skg_gcn {
  skg_plans* ps = nullptr;
  // CUDA graphs of the batched training step (gcn_dispatch); losses land in loss_scratch
  // and are copied to the caller's buffer after each replay
  GraphCache graphs;
  double* loss_scratch = nullptr;
  std::vector<const int32_t*> batch_seen;  // batch pointer last written per slot descriptor
  int L = 0, dtype = DT_F32;
  std::vector<int64_t> dims, ld;
  int64_t ld_max = 0, R = 0;
  int n_slots = 0;
  char* arena = nullptr;
  // layer-major activations: slot z of buffer X at X + z * R * ld(X) elements
  std::vector<char*> U, H;
  char* G0 = nullptr;
  char* G1 = nullptr;
  char* G2 = nullptr;  // G alternates G0 / G2 layer by layer (dW reads one, SpMM^T writes the other)
  // backward branch: dW_l and its slot reduction run on `side`, off the dX -> SpMM^T chain;
  // ev[l] forks it, ev[L + l] marks dW_l done, ev[2L] joins (captured as graph edges);
  // ev[2L + 1..3]: the weight split / label count branch at the start, the loss mean
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;
  // TF32 lo parts of the tensor-core GEMM operands (fp32 only): U_l, G, and the weights'
  // padded hi / lo copies (row stride ldw[l] = round4(d_{l+1}))
  std::vector<char*> Ulo, Wh, Wl;
  std::vector<int64_t> ldw;
  char* G0lo = nullptr;
  char* G2lo = nullptr;
  char* parts = nullptr;  // split-K partials of dW, one d_l x d_{l+1} block per slot
  int loss_kind = 0;      // 0: softmax cross-entropy (training.py:293-308); 1: multi-label BCE
  double pos_weight = 1.0;
  int64_t part_elems = 0;
  double* row_loss = nullptr;
  int32_t* nlab = nullptr;  // labelled rows per slot (softmax mean divisor)
  LayerDesc* d_layers = nullptr;      // [L][n_slots]
  SlotDesc* d_slots = nullptr;        // [n_slots]
  const int32_t** d_rows = nullptr;   // [L][n_slots] -> |S_{l+1}| scalars
};

// ------------------------------------------------------------------ small kernels
// symmetry check: w[j,i] exists and equals w[i,j] bitwise for every stored (i,j)
__global__ void k_check_symmetric(int64_t n, const int64_t* off, const int32_t* col,
                                  const double* w, int* bad) {
  SKG_PDL_PROLOGUE();
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    for (int64_t e = off[i] + threadIdx.x; e < off[i + 1]; e += blockDim.x) {
      int j = col[e];
      int64_t lo = off[j], hi = off[j + 1];
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (col[mid] < i) lo = mid + 1;
        else hi = mid;
      }
      if (lo >= off[j + 1] || col[lo] != i ||
          __double_as_longlong(w[lo]) != __double_as_longlong(w[e]))
        atomicExch(bad, 1);
    }
  }
}

// normalised-graph check: w[e] == 1.0/sqrt(d_i * d_j) bit for bit (graph.py:180-182)
__global__ void k_check_normalized(int64_t n, const int64_t* off, const int32_t* col,
                                   const double* w, double* degd, int* bad) {
  SKG_PDL_PROLOGUE();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    degd[i] = (double)(off[i + 1] - off[i]);
  __syncthreads();
}
__global__ void k_check_normalized2(int64_t n, const int64_t* off, const int32_t* col,
                                    const double* w, const double* degd, int* bad) {
  SKG_PDL_PROLOGUE();
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    for (int64_t e = off[i] + threadIdx.x; e < off[i + 1]; e += blockDim.x) {
      const double x = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(degd[i], degd[col[e]])));
      if (__double_as_longlong(x) != __double_as_longlong(w[e])) atomicExch(bad, 1);
    }
  }
}

__global__ void k_ids64_to_32(const int64_t* in, int64_t n, int32_t* out) {
  SKG_PDL_PROLOGUE();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

// ------------------------------------------------------------------ misc
extern "C" int skg_abi_version(void) { return 1; }

extern "C" int skg_profile_start(const char* kernel_name) {
  g_prof_target = kernel_name ? kernel_name : "";
  g_prof_pairs.clear();
  return SKG_OK;
}

extern "C" int skg_profile_stop(double* total_ms, int64_t* launches) {
  CK(cudaDeviceSynchronize());
  double tot = 0.0;
  for (auto& pr : g_prof_pairs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pr.a, pr.b);
    tot += ms;
    cudaEventDestroy(pr.a);
    cudaEventDestroy(pr.b);
  }
  *total_ms = tot;
  *launches = (int64_t)g_prof_pairs.size();
  g_prof_pairs.clear();
  g_prof_target.clear();
  return SKG_OK;
}

// per launch name: "name launches total_ms\n" lines into out (truncated to cap bytes)
extern "C" int skg_profile_table(char* out, int64_t cap) {
  ARG(out && cap > 0, "bad profile buffer");
  CK(cudaDeviceSynchronize());
  std::vector<std::string> order;
  std::unordered_map<std::string, std::pair<int64_t, double>> acc;
  for (auto& pr : g_prof_pairs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pr.a, pr.b);
    cudaEventDestroy(pr.a);
    cudaEventDestroy(pr.b);
    auto it = acc.find(pr.name);
    if (it == acc.end()) {
      order.push_back(pr.name);
      it = acc.emplace(pr.name, std::make_pair((int64_t)0, 0.0)).first;
    }
    it->second.first += 1;
    it->second.second += ms;
  }
  std::string txt;
  char line[512];
  for (auto& nm : order) {
    snprintf(line, sizeof(line), "%s %lld %.6f\n", nm.c_str(), (long long)acc[nm].first, acc[nm].second);
    txt += line;
  }
  g_prof_pairs.clear();
  g_prof_target.clear();
  const size_t n = std::min<size_t>(txt.size(), (size_t)cap - 1);
  memcpy(out, txt.data(), n);
  out[n] = 0;
  return SKG_OK;
}
extern "C" int skg_set_capture_only(int on) {
  g_capture_only = on ? 1 : 0;
  return SKG_OK;
}
extern "C" const char* skg_last_error(void) { return last_error(); }
extern "C" unsigned long long skg_kernel_launches(void) { return g_kernel_launches; }
extern "C" int skg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// ------------------------------------------------------------------ host RNG runtime
extern "C" int skg_spawn_pcg64(uint64_t master_seed, const char* const* label_reprs, int n_labels,
                               uint64_t out_state[4]) {
  ARG(n_labels >= 0 && out_state, "bad arguments");
  std::vector<std::string> labs;
  for (int i = 0; i < n_labels; ++i) labs.emplace_back(label_reprs[i]);
  Pcg64 g = spawn_pcg64(master_seed, labs);
  out_state[0] = (uint64_t)(g.state >> 64);
  out_state[1] = (uint64_t)g.state;
  out_state[2] = (uint64_t)(g.inc >> 64);
  out_state[3] = (uint64_t)g.inc;
  return SKG_OK;
}

static Pcg64 pcg_from(const uint64_t s[4], int has32, uint32_t u32) {
  Pcg64 g;
  g.state = ((u128)s[0] << 64) | s[1];
  g.inc = ((u128)s[2] << 64) | s[3];
  g.has32 = has32;
  g.u32 = u32;
  return g;
}

extern "C" int skg_choice_noreplace(const uint64_t state[4], int has32, uint32_t u32, int64_t pop,
                                    int64_t size, int64_t* out_idx) {
  ARG(pop >= 0 && size >= 0 && size <= pop, "Cannot take a larger sample than population when replace is False");
  Pcg64 g = pcg_from(state, has32, u32);
  choice_without_replacement(g, pop, size, out_idx);
  return SKG_OK;
}

extern "C" int skg_iteration_inputs(uint64_t master_seed, int64_t epoch, int64_t it, int64_t worker,
                                    const int64_t* train_w, int64_t n_train_w, int64_t batch_size,
                                    int64_t* out_batch, int64_t* out_len, uint64_t plan_state[4]) {
  ARG(n_train_w > 0, "worker has no training nodes");
  std::vector<std::string> lb = {repr_str("batch"), repr_int(epoch), repr_int(it), repr_int(worker)};
  Pcg64 g = spawn_pcg64(master_seed, lb);
  int64_t take = std::min(batch_size, n_train_w);
  std::vector<int64_t> idx(take);
  choice_without_replacement(g, n_train_w, take, idx.data());
  for (int64_t i = 0; i < take; ++i) out_batch[i] = train_w[idx[i]];
  std::sort(out_batch, out_batch + take);
  int64_t m = std::unique(out_batch, out_batch + take) - out_batch;
  *out_len = m;
  std::vector<std::string> lp = {repr_str("plan"), repr_int(epoch), repr_int(it), repr_int(worker)};
  Pcg64 p = spawn_pcg64(master_seed, lp);
  plan_state[0] = (uint64_t)(p.state >> 64);
  plan_state[1] = (uint64_t)p.state;
  plan_state[2] = (uint64_t)(p.inc >> 64);
  plan_state[3] = (uint64_t)p.inc;
  return SKG_OK;
}

// Persistent host thread pool for the per-iteration host work of whole look-ahead groups.
namespace {
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }
  // run fn(i) for i in [0, n) on up to `threads` workers (the caller takes part)
  void run(int n, int threads, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> one(call_);  // one group at a time
    threads = std::max(1, std::min(threads, n));
    // a forked child has none of the parent's workers: run inline there
    if (!th_.empty() && getpid() != pid_) threads = 1;
    if (threads == 1) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    std::unique_lock<std::mutex> lk(m_);
    ensure(threads - 1);
    job_ = &fn;
    n_ = n;
    next_.store(0);
    want_ = threads - 1;
    busy_ = 0;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    drain();
    lk.lock();
    done_.wait(lk, [&] { return busy_ == 0 && want_ == 0; });
    job_ = nullptr;
  }
  ~HostPool() {
    if (!th_.empty() && getpid() != pid_) {  // forked child: the threads are not ours
      for (auto& t : th_) t.detach();
      return;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }

 private:
  void ensure(int k) {
    if (th_.empty()) pid_ = getpid();
    while ((int)th_.size() < k) th_.emplace_back([this] { loop(); });
  }
  void drain() {
    for (int i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*job_)(i);
  }
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(m_);
    for (;;) {
      cv_.wait(lk, [&] { return stop_ || (gen_ != seen && want_ > 0); });
      if (stop_) return;
      seen = gen_;
      --want_;
      ++busy_;
      lk.unlock();
      drain();
      lk.lock();
      --busy_;
      if (busy_ == 0 && want_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_, call_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, want_ = 0, busy_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  pid_t pid_ = 0;
  std::atomic<int> next_{0};
};
}  // namespace

// skg_iteration_inputs for n worker-iterations at once (a Trainer look-ahead group): item i
// = (epochs[i], its[i], workers[i]) over the worker's training nodes train_ptrs[i] (length
// train_lens[i]); its batch is packed at out_batch[out_off[i] .. out_off[i + 1]) and its
// plan state at plan_states[4 i ..].  Items run on up to n_threads host threads; the
// results are those of n sequential skg_iteration_inputs calls.
extern "C" int skg_group_inputs(uint64_t master_seed, int n, const int64_t* epochs, const int64_t* its,
                                const int32_t* workers, const uint64_t* train_ptrs,
                                const int64_t* train_lens, int64_t batch_size, int64_t* out_batch,
                                int64_t* out_off, uint64_t* plan_states, int n_threads) {
  ARG(n >= 0 && batch_size >= 1 && epochs && its && workers && train_ptrs && train_lens && out_batch &&
          out_off && plan_states,
      "bad group inputs");
  for (int i = 0; i < n; ++i) ARG(train_lens[i] > 0, "worker has no training nodes");
  std::vector<int64_t> tmp((size_t)n * batch_size), len(n);
  HostPool::get().run(n, n_threads, [&](int i) {
    skg_iteration_inputs(master_seed, epochs[i], its[i], workers[i],
                         reinterpret_cast<const int64_t*>(train_ptrs[i]), train_lens[i], batch_size,
                         tmp.data() + (size_t)i * batch_size, &len[i], plan_states + 4 * (size_t)i);
  });
  out_off[0] = 0;
  for (int i = 0; i < n; ++i) {
    std::memcpy(out_batch + out_off[i], tmp.data() + (size_t)i * batch_size, sizeof(int64_t) * len[i]);
    out_off[i + 1] = out_off[i] + len[i];
  }
  return SKG_OK;
}

// ------------------------------------------------------------------ graph store
extern "C" int skg_ctx_create(int device, int64_t n, int64_t nnz, const int64_t* offsets,
                              const int32_t* neighbors, const double* weights, int32_t n_workers,
                              const int32_t* owner, skg_ctx** out) {
  ARG(out && offsets && n >= 0 && nnz >= 0, "bad arguments");
  ARG(n < (1LL << 31) - 64, "graphs with >= 2^31 nodes are not supported");
  ARG(offsets[0] == 0 && offsets[n] == nnz, "offsets must start at 0 and end at len(neighbors)");
  ARG(n_workers >= 1, "need at least one worker");
  CK(cudaSetDevice(device));
  skg_ctx* c = new skg_ctx();
  c->device = device;
  c->n = n;
  c->nnz = nnz;
  c->n_workers = n_workers;
  CK(cudaMalloc(&c->d_off, sizeof(int64_t) * (n + 1)));
  CK(cudaMalloc(&c->d_col, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  CK(cudaMalloc(&c->d_w, sizeof(double) * std::max<int64_t>(nnz, 1)));
  CK(cudaMalloc(&c->d_owner, sizeof(int32_t) * std::max<int64_t>(n, 1)));
  CK(cudaMemcpy(c->d_off, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  if (nnz) {
    CK(cudaMemcpy(c->d_col, neighbors, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_w, weights, sizeof(double) * nnz, cudaMemcpyHostToDevice));
  }
  if (n) {
    if (owner) CK(cudaMemcpy(c->d_owner, owner, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    else CK(cudaMemset(c->d_owner, 0, sizeof(int32_t) * n));
  }
  // degree bound table for arena sizing
  std::vector<int64_t> deg(n);
  for (int64_t i = 0; i < n; ++i) deg[i] = offsets[i + 1] - offsets[i];
  std::sort(deg.begin(), deg.end(), std::greater<int64_t>());
  c->deg_desc_prefix.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) c->deg_desc_prefix[i + 1] = c->deg_desc_prefix[i] + deg[i];
  // symmetric weights (every normalised graph): the CSC used by pull passes is the CSR
  int* d_bad;
  CK(cudaMalloc(&d_bad, sizeof(int)));
  CK(cudaMemset(d_bad, 0, sizeof(int)));
  if (n) k_check_symmetric<<<std::min<int64_t>(n, 65535), 256>>>(n, c->d_off, c->d_col, c->d_w, d_bad);
  int bad = 0;
  CK(cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost));
  c->symmetric = !bad;
  CK(cudaMalloc(&c->d_degd, sizeof(double) * std::max<int64_t>(n, 1)));
  CK(cudaMemset(d_bad, 0, sizeof(int)));
  if (n) {
    k_check_normalized<<<std::min<int64_t>((n + 255) / 256, 4096), 256>>>(n, c->d_off, c->d_col, c->d_w, c->d_degd, d_bad);
    k_check_normalized2<<<std::min<int64_t>(n, 65535), 256>>>(n, c->d_off, c->d_col, c->d_w, c->d_degd, d_bad);
  }
  CK(cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost));
  c->normalized = (n > 0) && !bad;
  if (getenv("SKG_STORED_WEIGHTS")) c->normalized = false;  // experiment: read w, never recompute
  cudaFree(d_bad);
  // the fused range expand (sampler.cu k_lad_range) serves normalised graphs; its
  // graph-static range-start table is built per range size when a plan set first needs it
  c->fr_ok = c->normalized && n >= 1;
  if (!c->symmetric) {  // host counting sort by column (rows ascending within a column)
    std::vector<int64_t> toff(n + 1, 0);
    for (int64_t e = 0; e < nnz; ++e) toff[neighbors[e] + 1]++;
    for (int64_t i = 0; i < n; ++i) toff[i + 1] += toff[i];
    std::vector<int64_t> fill(toff.begin(), toff.end() - 1);
    std::vector<int32_t> trow(std::max<int64_t>(nnz, 1));
    std::vector<double> tw(std::max<int64_t>(nnz, 1));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t e = offsets[i]; e < offsets[i + 1]; ++e) {
        int64_t p = fill[neighbors[e]]++;
        trow[p] = (int32_t)i;
        tw[p] = weights[e];
      }
    CK(cudaMalloc(&c->d_toff, sizeof(int64_t) * (n + 1)));
    CK(cudaMalloc(&c->d_trow, sizeof(int32_t) * trow.size()));
    CK(cudaMalloc(&c->d_tw, sizeof(double) * tw.size()));
    CK(cudaMemcpy(c->d_toff, toff.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_trow, trow.data(), sizeof(int32_t) * trow.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_tw, tw.data(), sizeof(double) * tw.size(), cudaMemcpyHostToDevice));
  }
  CK(cudaDeviceSynchronize());
  *out = c;
  return SKG_OK;
}

extern "C" int skg_ctx_destroy(skg_ctx* c) {
  if (!c) return SKG_OK;
  cudaSetDevice(c->device);
  cudaFree(c->d_off);
  cudaFree(c->d_col);
  cudaFree(c->d_w);
  cudaFree(c->d_owner);
  cudaFree(c->d_toff);
  cudaFree(c->d_trow);
  cudaFree(c->d_tw);
  cudaFree(c->d_degd);
  for (auto& kv : c->rstarts) cudaFree(kv.second);
  cudaFree(c->d_x);
  cudaFree(c->d_labels);
  cudaFree(c->d_ymulti);
  cudaFree(c->d_shards);
  cudaFree(c->d_node_rank);
  cudaFree(c->d_node_row);
  for (void* p : c->shards_owned) cudaFree(p);
  delete c;
  return SKG_OK;
}

extern "C" int skg_ctx_set_features(skg_ctx* c, int dtype, int64_t dim, int64_t n_rows,
                                    const void* host_rows) {
  if (c) ++c->gen;
  ARG(c && (dtype == DT_F32 || dtype == DT_F64) && dim > 0 && n_rows >= 0, "bad feature arguments");
  CK(cudaSetDevice(c->device));
  const size_t es = dtype == DT_F32 ? 4 : 8;
  cudaFree(c->d_x);
  c->d_x = nullptr;
  c->F = dim;
  c->ldx = round4(dim);
  c->dtype = dtype;
  c->x_rows = n_rows;
  c->xbits = 0;
  CK(cudaMalloc(&c->d_x, es * c->ldx * std::max<int64_t>(n_rows, 1)));
  CK(cudaMemset(c->d_x, 0, es * c->ldx * std::max<int64_t>(n_rows, 1)));
  if (n_rows)
    CK(cudaMemcpy2D(c->d_x, es * c->ldx, host_rows, es * dim, es * dim, n_rows, cudaMemcpyHostToDevice));
  // single-rank default map: shard 0 = all rows, row = node
  cudaFree(c->d_shards);
  CK(cudaMalloc(&c->d_shards, sizeof(uint64_t)));
  uint64_t p = (uint64_t)c->d_x;
  CK(cudaMemcpy(c->d_shards, &p, sizeof(uint64_t), cudaMemcpyHostToDevice));
  c->n_ranks = 1;
  cudaFree(c->d_node_rank);
  cudaFree(c->d_node_row);
  c->d_node_rank = nullptr;
  c->d_node_row = nullptr;
  return SKG_OK;
}

// Multi-hot (0 / 1) features bit-packed on the device: row i is words_per_row 32-bit words,
// feature c at bit (c & 31) of word (c >> 5); expanded to 0 / 1 in the compute dtype by the
// layer-0 SpMM (the same products as dense 0 / 1 rows, 32x fewer feature bytes).
extern "C" int skg_ctx_set_features_bits(skg_ctx* c, int dtype, int64_t dim, int64_t n_rows,
                                         const uint32_t* host_words, int64_t words_per_row) {
  if (c) ++c->gen;
  ARG(c && (dtype == DT_F32 || dtype == DT_F64) && dim > 0 && n_rows >= 0 &&
          words_per_row >= (dim + 31) / 32 && (host_words || !n_rows),
      "bad bit-packed feature arguments");
  CK(cudaSetDevice(c->device));
  cudaFree(c->d_x);
  c->d_x = nullptr;
  c->F = dim;
  c->ldx = (((dim + 31) / 32) + 3) / 4 * 4;  // words, padded to 16 bytes
  c->dtype = dtype;
  c->x_rows = n_rows;
  c->xbits = 1;
  CK(cudaMalloc(&c->d_x, 4 * c->ldx * std::max<int64_t>(n_rows, 1)));
  CK(cudaMemset(c->d_x, 0, 4 * c->ldx * std::max<int64_t>(n_rows, 1)));
  if (n_rows)
    CK(cudaMemcpy2D(c->d_x, 4 * c->ldx, host_words, 4 * words_per_row, 4 * ((dim + 31) / 32), n_rows,
                    cudaMemcpyHostToDevice));
  cudaFree(c->d_shards);
  CK(cudaMalloc(&c->d_shards, sizeof(uint64_t)));
  uint64_t p = (uint64_t)c->d_x;
  CK(cudaMemcpy(c->d_shards, &p, sizeof(uint64_t), cudaMemcpyHostToDevice));
  c->n_ranks = 1;
  cudaFree(c->d_node_rank);
  cudaFree(c->d_node_row);
  c->d_node_rank = nullptr;
  c->d_node_row = nullptr;
  return SKG_OK;
}

extern "C" int skg_ctx_set_feature_map(skg_ctx* c, int n_ranks, const uint64_t* shard_ptrs,
                                       const int32_t* node_rank, const int32_t* node_row) {
  if (c) ++c->gen;
  ARG(c && n_ranks >= 1 && shard_ptrs && node_rank && node_row, "bad feature map");
  CK(cudaSetDevice(c->device));
  cudaFree(c->d_shards);
  cudaFree(c->d_node_rank);
  cudaFree(c->d_node_row);
  CK(cudaMalloc(&c->d_shards, sizeof(uint64_t) * n_ranks));
  CK(cudaMemcpy(c->d_shards, shard_ptrs, sizeof(uint64_t) * n_ranks, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&c->d_node_rank, sizeof(int32_t) * c->n));
  CK(cudaMalloc(&c->d_node_row, sizeof(int32_t) * c->n));
  CK(cudaMemcpy(c->d_node_rank, node_rank, sizeof(int32_t) * c->n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_node_row, node_row, sizeof(int32_t) * c->n, cudaMemcpyHostToDevice));
  c->n_ranks = n_ranks;
  return SKG_OK;
}

extern "C" int skg_ctx_shard_upload(skg_ctx* c, const void* host_rows, int64_t n_rows,
                                    uint64_t* out_dev_ptr) {
  ARG(c && c->d_x && n_rows >= 0 && out_dev_ptr, "set features before uploading shards");
  CK(cudaSetDevice(c->device));
  // bit-packed features: host rows are ceil(F / 32) words each
  const size_t es = c->xbits ? 4 : c->dtype == DT_F32 ? 4 : 8;
  const int64_t in_elems = c->xbits ? (c->F + 31) / 32 : c->F;
  void* p = nullptr;
  CK(cudaMalloc(&p, es * c->ldx * std::max<int64_t>(n_rows, 1)));
  CK(cudaMemset(p, 0, es * c->ldx * std::max<int64_t>(n_rows, 1)));
  if (n_rows)
    CK(cudaMemcpy2D(p, es * c->ldx, host_rows, es * in_elems, es * in_elems, n_rows, cudaMemcpyHostToDevice));
  c->shards_owned.push_back(p);
  *out_dev_ptr = (uint64_t)p;
  return SKG_OK;
}

extern "C" int skg_ctx_feature_ptr(skg_ctx* c, uint64_t* out_ptr, int64_t* out_ld) {
  ARG(c, "null ctx");
  *out_ptr = (uint64_t)c->d_x;
  *out_ld = c->ldx;
  return SKG_OK;
}

extern "C" int skg_ctx_set_labels(skg_ctx* c, const int64_t* labels) {
  if (c) ++c->gen;
  ARG(c && labels, "bad labels");
  CK(cudaSetDevice(c->device));
  std::vector<int32_t> l32(c->n);
  for (int64_t i = 0; i < c->n; ++i) l32[i] = (int32_t)labels[i];
  cudaFree(c->d_labels);
  CK(cudaMalloc(&c->d_labels, sizeof(int32_t) * std::max<int64_t>(c->n, 1)));
  if (c->n) CK(cudaMemcpy(c->d_labels, l32.data(), sizeof(int32_t) * c->n, cudaMemcpyHostToDevice));
  return SKG_OK;
}

// multi-hot targets for the multi-label (BCE) loss: n x words uint64, bit k of word k/64
extern "C" int skg_ctx_set_multilabels(skg_ctx* c, const uint64_t* words, int32_t n_classes) {
  if (c) ++c->gen;
  ARG(c && words && n_classes >= 1, "bad multi-labels");
  CK(cudaSetDevice(c->device));
  const int32_t nw = (n_classes + 63) / 64;
  cudaFree(c->d_ymulti);
  CK(cudaMalloc(&c->d_ymulti, sizeof(uint64_t) * nw * std::max<int64_t>(c->n, 1)));
  if (c->n) CK(cudaMemcpy(c->d_ymulti, words, sizeof(uint64_t) * nw * c->n, cudaMemcpyHostToDevice));
  c->y_words = nw;
  c->y_classes = n_classes;
  return SKG_OK;
}

extern "C" int skg_ctx_set_owner(skg_ctx* c, int32_t n_workers, const int32_t* owner) {
  if (c) ++c->gen;
  ARG(c && owner && n_workers >= 1, "bad owner map");
  CK(cudaSetDevice(c->device));
  for (int64_t i = 0; i < c->n; ++i)
    if (owner[i] < 0 || owner[i] >= n_workers) {
      set_error("owner id out of range");
      return SKG_ERR_ARG;
    }
  if (c->n) CK(cudaMemcpy(c->d_owner, owner, sizeof(int32_t) * c->n, cudaMemcpyHostToDevice));
  c->n_workers = n_workers;
  return SKG_OK;
}

extern "C" int skg_ctx_info(skg_ctx* c, int64_t out[8]) {
  ARG(c, "null ctx");
  out[0] = c->n;
  out[1] = c->nnz;
  out[2] = c->symmetric;
  out[3] = c->ldx;
  out[4] = c->F;
  out[5] = c->dtype;
  out[6] = c->device;
  out[7] = c->n_ranks | ((int64_t)c->normalized << 32) | ((int64_t)c->xbits << 33);
  return SKG_OK;
}

extern "C" int skg_ipc_handle(uint64_t dev_ptr, uint8_t out_handle[64]) {
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, (void*)dev_ptr));
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(out_handle, &h, 64);
  return SKG_OK;
}
extern "C" int skg_ipc_open(const uint8_t handle[64], uint64_t* out_dev_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *out_dev_ptr = (uint64_t)p;
  return SKG_OK;
}
extern "C" int skg_ipc_close(uint64_t dev_ptr) {
  CK(cudaIpcCloseMemHandle((void*)dev_ptr));
  return SKG_OK;
}

// ------------------------------------------------------------------ plan arenas
struct Carver {
  size_t off = 0;
  std::vector<std::pair<void**, size_t>> items;
  template <typename T>
  void add(T*& p, size_t count) {
    items.push_back({reinterpret_cast<void**>(&p), off});
    off += (count * sizeof(T) + 255) / 256 * 256;
  }
  void bind(char* base) {
    for (auto& it : items) *it.first = base + it.second;
  }
};

extern "C" int skg_plans_create(skg_ctx* c, int kind, int n_slots, int L, int64_t budget,
                                int64_t max_batch, skg_plans** out) {
  ARG(c && out && n_slots >= 1 && L >= 1 && budget >= 1, "bad plan-set arguments");
  ARG(kind == KIND_LADIES || kind == KIND_SAINT, "unknown plan kind");
  ARG(budget < (1LL << 20), "budget too large for the device sampler");
  CK(cudaSetDevice(c->device));
  skg_plans* ps = new skg_plans();
  ps->ctx = c;
  ps->kind = kind;
  ps->n_slots = n_slots;
  ps->L = L;
  ps->budget = budget;
  ps->max_batch = std::max<int64_t>(max_batch, 1);
  const int64_t n = c->n;
  const int n_words = (int)((n + 31) / 32);
  int64_t cap_rows, cap_cand, cap_pairs, cap_batch;
  if (kind == KIND_LADIES) {
    cap_rows = std::min<int64_t>(std::max<int64_t>(ps->max_batch, budget), std::max<int64_t>(n, 1));
    cap_pairs = std::max<int64_t>(c->edge_bound(cap_rows), 1);
    cap_cand = std::max<int64_t>(std::min<int64_t>(n, cap_pairs), 1);
    cap_batch = ps->max_batch;
  } else {
    cap_rows = std::min<int64_t>(budget, std::max<int64_t>(n, 1));
    cap_pairs = std::max<int64_t>(c->edge_bound(cap_rows), 1);
    cap_cand = std::max<int64_t>(n, 1);
    cap_batch = 1;
  }
  // per-layer arrays are strided by cap_cand: a multiple of 16 keeps every layer's norm and
  // flag rows aligned for the vector loads of the pairwise leaves (k_pw_leaves)
  cap_cand = (cap_cand + 15) / 16 * 16;
  ARG(cap_pairs < (1LL << 31) && cap_cand < (1LL << 31), "plan capacity exceeds int32 indexing");
  // LADIES keeps upper-row ranks in 16-bit slots / counters
  ARG(kind != KIND_LADIES || cap_rows < 65535, "LADIES batch / budget must be below 65535");
  ps->cap_rows = (int)cap_rows;
  ps->cap_cand = (int)cap_cand;
  ps->cap_pairs = cap_pairs;
  ps->cap_batch = (int)cap_batch;
  // fused range expand (sampler.cu k_lad_range): normalised graphs of <= kMaxFR ranges;
  // SKG_EXPAND=ranges|global (or SKG_GLOBAL_EXPAND) selects the older expand kernels
  {
    const char* ex = getenv("SKG_EXPAND");
    const bool off = getenv("SKG_GLOBAL_EXPAND") || (ex && std::string(ex) != "fused");
    ps->n_fr = 0;
    if (kind == KIND_LADIES && c->fr_ok && !off && cap_rows <= kFusedMaxRows) {
      const int max_upper = L > 1 ? (int)std::max<int64_t>(cap_batch, std::min<int64_t>(budget, cap_cand))
                                  : (int)cap_batch;
      int nfr = 0;
      const int fr = choose_fr(n, n_slots, max_upper, &nfr);
      if (fr > 0 && nfr >= 1 && nfr <= kMaxFR) {
        auto it = c->rstarts.find(fr);
        if (it == c->rstarts.end()) {
          int32_t* tab = nullptr;
          CK(cudaMalloc(&tab, sizeof(int32_t) * (size_t)n * (nfr + 1)));
          GraphDev g = c->gdev();
          g.fr_size = fr;
          int rc = launch_build_rstart(g, tab, nfr);
          if (rc) {
            cudaFree(tab);
            return rc;
          }
          CK(cudaDeviceSynchronize());
          it = c->rstarts.emplace(fr, tab).first;
        }
        ps->n_fr = nfr;
        ps->fr_size = fr;
        if (getenv("SKG_DEBUG_FR"))
          fprintf(stderr, "skg: fused expand %d ranges x %d nodes for %d plans\n", nfr, fr, n_slots);
        ps->rstart = it->second;
      }
    }
  }
  const int Ls = kind == KIND_LADIES ? L : 1;
  int pw = 0;
  while (cap_cand > (112LL << pw)) ++pw;
  const int cap_slots = std::max(1 << pw, kPwSub);
  const int cap_chunks = (int)((cap_cand + kChunk - 1) / kChunk);
  const int cap_supers = (int)((cap_cand + kSuper - 1) / kSuper);
  const int cap_tiles = (int)std::max<int64_t>((n_words + kTileWords - 1) / kTileWords,
                                               (cap_cand + kTileCand - 1) / kTileCand) + 1;
  ps->h.resize(n_slots);
  // per-slot scalars (zeroed per sampling call): err, starvation, draws, counters
  Carver scal;
  std::vector<int32_t*> errs(n_slots), starv(n_slots), ctrs(n_slots);
  std::vector<int64_t*> draws(n_slots);
  std::vector<unsigned long long*> looks(n_slots);
  for (int s = 0; s < n_slots; ++s) {
    scal.add(errs[s], 1);
    scal.add(starv[s], 1);
    scal.add(ctrs[s], 8);
    scal.add(draws[s], 1);
    scal.add(looks[s], ps->n_fr ? (size_t)L * kMaxFR : 1);
  }
  ps->scal_bytes = scal.off;
  Carver cv;
  for (int s = 0; s < n_slots; ++s) {
    PlanDev& P = ps->h[s];
    memset(&P, 0, sizeof(P));
    P.cap_rows = (int)cap_rows;
    P.cap_cand = (int)cap_cand;
    P.cap_pairs = cap_pairs;
    P.cap_chunks = cap_chunks;
    P.cap_supers = cap_supers;
    P.cap_slots = cap_slots;
    P.cap_tiles = cap_tiles;
    cv.add(P.bitmap, n_words);
    cv.add(P.sbitmap, n_words);
    cv.add(P.bitmap1, (size_t)(n_words + 31) / 32);
    cv.add(P.dirty, 1);
    cv.add(P.cnt_pack, ps->n_fr ? 1 : (size_t)(n / 2 + 1));
    const bool lad = kind == KIND_LADIES, stw = lad && !c->normalized;
    cv.add(P.slots, lad && !ps->n_fr ? (size_t)std::max<int64_t>(n, 1) * kSlots : 4);
    cv.add(P.cslots, lad && c->normalized ? cap_cand : 1);
    cv.add(P.slotw, stw ? (size_t)std::max<int64_t>(n, 1) * kSlots : 1);
    cv.add(P.ov, lad ? cap_pairs : 1);
    cv.add(P.ovw, stw ? cap_pairs : 1);
    cv.add(P.hidx, lad ? (size_t)std::max<int64_t>(n, 1) : 1);
    cv.add(P.hoff, lad ? cap_cand : 1);
    cv.add(P.hfill, lad ? cap_cand : 1);
    cv.add(P.hbuf, lad ? cap_pairs : 1);
    cv.add(P.hbufw, stw ? cap_pairs : 1);
    cv.add(P.heavy, lad ? cap_cand : 1);
    cv.add(P.huge, lad ? cap_cand : 1);
    cv.add(P.updeg, lad ? cap_rows : 1);
    cv.add(P.row_any, lad ? cap_rows : 1);
    cv.add(P.cand_cnt, lad ? cap_cand : 1);
    cv.add(P.pair_off, cap_rows + 1);
    cv.add(P.word_prefix, n_words);
    cv.add(P.tile_a, cap_tiles);
    cv.add(P.pw_val, cap_slots);
    cv.add(P.pw_lvl, cap_slots);
    cv.add(P.chunk_sum, cap_chunks);
    cv.add(P.chunk_approx, cap_chunks);
    cv.add(P.chunk_map, 2 * (size_t)cap_chunks);
    cv.add(P.chunk_e, cap_chunks);
    cv.add(P.chunk_mode, cap_chunks);
    cv.add(P.chunk_start, cap_chunks);
    cv.add(P.super_map, 2 * (size_t)cap_supers);
    cv.add(P.super_e, cap_supers);
    cv.add(P.super_mode, cap_supers);
    cv.add(P.super_start, cap_supers);
    cv.add(P.cdf, cap_cand);
    cv.add(P.draw_idx, budget);
    cv.add(P.cand, kind == KIND_LADIES ? (size_t)Ls * cap_cand : 1);
    cv.add(P.norm, (size_t)Ls * cap_cand);
    cv.add(P.is_local, (size_t)Ls * cap_cand);
    cv.add(P.nodes, (size_t)Ls * cap_rows);
    cv.add(P.samp_rank, (size_t)Ls * cap_rows);
    cv.add(P.p, (size_t)Ls * cap_rows);
    cv.add(P.indptr, (size_t)Ls * (cap_rows + 1));
    cv.add(P.indices, (size_t)Ls * cap_pairs);
    cv.add(P.val, (size_t)Ls * cap_pairs);
    cv.add(P.tindptr, (size_t)Ls * (cap_rows + 1));
    cv.add(P.tindices, (size_t)Ls * cap_pairs);
    cv.add(P.tval, (size_t)Ls * cap_pairs);
    cv.add(P.stat, L);
  }
  int32_t* d_batch = nullptr;
  cv.add(d_batch, (size_t)n_slots * cap_batch);
  cudaError_t e1 = cudaMalloc(&ps->arena, cv.off);
  if (e1 != cudaSuccess) {
    set_error(std::string("plan arena (") + std::to_string(cv.off >> 20) + " MiB): " +
              cudaGetErrorString(e1));
    delete ps;
    return SKG_ERR_CUDA;
  }
  cv.bind(ps->arena);
  ps->d_batch = d_batch;
  CK(cudaMalloc(&ps->d_scal, scal.off));
  scal.bind(ps->d_scal);
  CK(cudaMemset(ps->arena, 0, cv.off));
  CK(cudaMemset(ps->d_scal, 0, scal.off));
  for (int s = 0; s < n_slots; ++s) {
    PlanDev& P = ps->h[s];
    P.err = errs[s];
    P.starvation = starv[s];
    P.counters = ctrs[s];
    P.draws_consumed = draws[s];
    P.look = looks[s];
    P.n_fr = ps->n_fr;
    P.kind = kind;
    P.n_layers = L;
    P.budget = budget;
  }
  CK(cudaMalloc(&ps->d_plans, sizeof(PlanDev) * n_slots));
  CK(cudaMemcpy(ps->d_plans, ps->h.data(), sizeof(PlanDev) * n_slots, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&ps->d_sticky, sizeof(int32_t)));
  CK(cudaMemset(ps->d_sticky, 0, sizeof(int32_t)));
  *out = ps;
  return SKG_OK;
}

extern "C" int skg_plans_destroy(skg_plans* ps) {
  if (!ps) return SKG_OK;
  cudaSetDevice(ps->ctx->device);
  ps->graphs.clear();
  if (ps->graphs.cap) cudaStreamDestroy(ps->graphs.cap);
  if (ps->up_ev) {
    cudaEventSynchronize(ps->up_ev);
    cudaEventDestroy(ps->up_ev);
  }
  if (ps->h_pin) cudaFreeHost(ps->h_pin);
  if (ps->hb_pin) cudaFreeHost(ps->hb_pin);
  if (ps->hu_pin) cudaFreeHost(ps->hu_pin);
  cudaFree(ps->d_unif);
  cudaFree(ps->arena);
  cudaFree(ps->d_scal);
  cudaFree(ps->d_plans);
  cudaFree(ps->d_sticky);
  cudaFree(ps->d_train);
  cudaFree(ps->d_train_norm);
  cudaFree(ps->d_train_bitmap);
  for (auto p : ps->d_local) cudaFree(p);
  for (auto p : ps->d_local_norm) cudaFree(p);
  delete ps;
  return SKG_OK;
}

static int status_from_err(int err) {
  if (err & EB_NOT_ADJACENT) {
    set_error("candidates not adjacent to s_l");
    return SKG_ERR_NOT_ADJACENT;
  }
  if (err & EB_NO_LABELS) {
    set_error("batch contains no labeled nodes");
    return SKG_ERR_NO_LABELS;
  }
  if (err & EB_CAPACITY) {
    set_error("plan arena capacity exceeded");
    return SKG_ERR_CAPACITY;
  }
  return SKG_OK;
}

static int ladies_sample(skg_plans* ps, int n, const int32_t* workers, const int64_t* batch_off,
                         const int64_t* batch_ids, int mode, double D, double min_scale,
                         const skg_rng* rngs, const uint64_t* rng, void* stream) {
  ARG(ps && ps->kind == KIND_LADIES, "not a LADIES plan set");
  ARG(n >= 1 && n <= ps->n_slots, "slot count out of range");
  ARG(mode >= 0 && mode <= 2, "unknown mode");
  skg_ctx* c = ps->ctx;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = staging_ready(ps);
  if (rc) return rc;
  int32_t* hb = ps->hb_pin;
  for (int i = 0; i < n; ++i) {
    int64_t len = batch_off[i + 1] - batch_off[i];
    if (len <= 0) {
      set_error("empty batch");
      return SKG_ERR_EMPTY;
    }
    ARG(len <= ps->cap_batch, "batch larger than the plan set's max_batch");
    ARG(workers[i] >= 0 && workers[i] < c->n_workers, "worker id out of range");
    for (int64_t k = 0; k < len; ++k) {
      int64_t v = batch_ids[batch_off[i] + k];
      if (v < 0 || v >= c->n) {
        set_error("node id out of range for this graph");
        return SKG_ERR_ARG;
      }
      if (k && v <= batch_ids[batch_off[i] + k - 1]) {
        set_error("node set must be strictly increasing");
        return SKG_ERR_ARG;
      }
      hb[(size_t)i * ps->cap_batch + k] = (int32_t)v;
    }
    PlanDev& P = ps->h[i];
    P.worker = workers[i];
    P.mode = mode;
    P.D = D;
    P.min_scale = min_scale;
    rc = set_rng(ps, P, i, rngs, rng);
    if (rc) return rc;
    P.batch_len = (int32_t)len;
    P.batch = ps->d_batch + (size_t)i * ps->cap_batch;
    P.cand_norm = nullptr;
  }
  rc = upload_plans(ps, n, (size_t)n * ps->cap_batch, st);
  if (rc) return rc;
  CK(cudaMemsetAsync(ps->d_scal, 0, ps->scal_bytes, st));
  const int max_upper = ps->L > 1 ? std::max<int>(ps->cap_batch, (int)std::min<int64_t>(ps->budget, ps->cap_cand))
                                  : ps->cap_batch;
  return run_ladies(ps, n, max_upper, st);
}

extern "C" int skg_ladies_sample(skg_plans* ps, int n, const int32_t* workers,
                                 const int64_t* batch_off, const int64_t* batch_ids, int mode,
                                 double D, double min_scale, const uint64_t* rng, void* stream) {
  ARG(rng, "bad arguments");
  return ladies_sample(ps, n, workers, batch_off, batch_ids, mode, D, min_scale, nullptr, rng, stream);
}

extern "C" int skg_ladies_sample_rng(skg_plans* ps, int n, const int32_t* workers,
                                     const int64_t* batch_off, const int64_t* batch_ids, int mode,
                                     double D, double min_scale, const skg_rng* rngs, void* stream) {
  ARG(rngs, "bad arguments");
  return ladies_sample(ps, n, workers, batch_off, batch_ids, mode, D, min_scale, rngs, nullptr, stream);
}

extern "C" int skg_ladies_sample_device(skg_plans* ps, int n, const int32_t* workers,
                                        const int32_t* batch_len, uint64_t d_batch,
                                        int64_t batch_stride, int mode, double D, double min_scale,
                                        const uint64_t* rng, void* stream) {
  ARG(ps && ps->kind == KIND_LADIES, "not a LADIES plan set");
  ARG(n >= 1 && n <= ps->n_slots && d_batch, "bad arguments");
  skg_ctx* c = ps->ctx;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = staging_ready(ps);
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    if (batch_len[i] <= 0) {
      set_error("empty batch");
      return SKG_ERR_EMPTY;
    }
    ARG(batch_len[i] <= ps->cap_batch, "batch larger than the plan set's max_batch");
    ARG(workers[i] >= 0 && workers[i] < c->n_workers, "worker id out of range");
    PlanDev& P = ps->h[i];
    P.worker = workers[i];
    P.mode = mode;
    P.D = D;
    P.min_scale = min_scale;
    rc = set_rng(ps, P, i, nullptr, rng);
    if (rc) return rc;
    P.batch_len = batch_len[i];
    P.batch = reinterpret_cast<const int32_t*>(d_batch) + (size_t)i * batch_stride;
    P.cand_norm = nullptr;
  }
  rc = upload_plans(ps, n, 0, st);
  if (rc) return rc;
  CK(cudaMemsetAsync(ps->d_scal, 0, ps->scal_bytes, st));
  const int max_upper = ps->L > 1 ? std::max<int>(ps->cap_batch, (int)std::min<int64_t>(ps->budget, ps->cap_cand))
                                  : ps->cap_batch;
  return run_ladies(ps, n, max_upper, st);
}

// column_norms(g, rows, candidates) (graph.py:198-220) by the pull formulation: for each
// candidate j an ordered fold over column j (i ascending, == the np.add.at order) of w_ij^2
// for i in `rows`.  Used for large row sets (GraphSAINT's training set), where the push
// (LADIES expand) form would need a plan per call.
extern "C" int skg_column_norms_pull(skg_ctx* c, const int64_t* rows, int64_t n_rows,
                                     const int64_t* cand, int64_t n_cand, double* out) {
  ARG(c && rows && cand && out && n_rows >= 1 && n_cand >= 0, "bad column-norm arguments");
  ARG(n_rows < (1LL << 31) && n_cand < (1LL << 31), "node set too large");
  CK(cudaSetDevice(c->device));
  if (n_cand == 0) return SKG_OK;
  std::vector<int32_t> r32(n_rows), c32(n_cand);
  for (int64_t i = 0; i < n_rows; ++i) {
    ARG(rows[i] >= 0 && rows[i] < c->n, "node id out of range for this graph");
    ARG(i == 0 || rows[i] > rows[i - 1], "node set must be strictly increasing");
    r32[i] = (int32_t)rows[i];
  }
  for (int64_t i = 0; i < n_cand; ++i) {
    ARG(cand[i] >= 0 && cand[i] < c->n, "node id out of range for this graph");
    ARG(i == 0 || cand[i] > cand[i - 1], "node set must be strictly increasing");
    c32[i] = (int32_t)cand[i];
  }
  const int n_words = (int)((c->n + 31) / 32);
  int32_t *d_rows = nullptr, *d_cand = nullptr, *d_err = nullptr;
  uint32_t* d_bm = nullptr;
  double* d_out = nullptr;
  CK(cudaMalloc(&d_rows, 4 * n_rows));
  CK(cudaMalloc(&d_cand, 4 * n_cand));
  CK(cudaMalloc(&d_bm, 4 * (size_t)n_words));
  CK(cudaMalloc(&d_out, 8 * n_cand));
  CK(cudaMalloc(&d_err, 4));
  CK(cudaMemset(d_err, 0, 4));
  CK(cudaMemcpy(d_rows, r32.data(), 4 * n_rows, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cand, c32.data(), 4 * n_cand, cudaMemcpyHostToDevice));
  launch_set_bitmap(d_rows, (int32_t)n_rows, d_bm, n_words, 0);
  int rc = launch_pull_norms(c->gdev(), d_cand, (int32_t)n_cand, d_bm, d_out, d_err, 0);
  int err = 0;
  cudaError_t e = cudaDeviceSynchronize();
  if (!rc && e == cudaSuccess) {
    cudaMemcpy(out, d_out, 8 * n_cand, cudaMemcpyDeviceToHost);
    cudaMemcpy(&err, d_err, 4, cudaMemcpyDeviceToHost);
  }
  cudaFree(d_rows);
  cudaFree(d_cand);
  cudaFree(d_bm);
  cudaFree(d_out);
  cudaFree(d_err);
  if (rc) return rc;
  if (e != cudaSuccess) {
    set_error(std::string("column norms: ") + cudaGetErrorString(e));
    return SKG_ERR_CUDA;
  }
  if (err & EB_NOT_ADJACENT) {
    set_error("candidates not adjacent to s_l");
    return SKG_ERR_NOT_ADJACENT;
  }
  return SKG_OK;
}

extern "C" int skg_saint_set_candidates(skg_plans* ps, const int64_t* train, int64_t n_train,
                                        int precompute, void* stream) {
  ARG(ps && ps->kind == KIND_SAINT, "not a SAINT plan set");
  ARG(n_train >= 1, "empty training node set");
  skg_ctx* c = ps->ctx;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int32_t> t32(n_train);
  for (int64_t i = 0; i < n_train; ++i) {
    ARG(train[i] >= 0 && train[i] < c->n, "node id out of range for this graph");
    ARG(i == 0 || train[i] > train[i - 1], "node set must be strictly increasing");
    t32[i] = (int32_t)train[i];
  }
  cudaFree(ps->d_train);
  cudaFree(ps->d_train_norm);
  cudaFree(ps->d_train_bitmap);
  for (auto p : ps->d_local) cudaFree(p);
  for (auto p : ps->d_local_norm) cudaFree(p);
  ps->d_local.assign(c->n_workers, nullptr);
  ps->d_local_norm.assign(c->n_workers, nullptr);
  ps->n_local.assign(c->n_workers, 0);
  ps->local_norm_ready.assign(c->n_workers, false);
  ps->n_train = n_train;
  const int n_words = (int)((c->n + 31) / 32);
  CK(cudaMalloc(&ps->d_train, sizeof(int32_t) * n_train));
  CK(cudaMalloc(&ps->d_train_norm, sizeof(double) * n_train));
  CK(cudaMalloc(&ps->d_train_bitmap, sizeof(uint32_t) * n_words));
  CK(cudaMemcpyAsync(ps->d_train, t32.data(), sizeof(int32_t) * n_train, cudaMemcpyHostToDevice, st));
  launch_set_bitmap(ps->d_train, (int32_t)n_train, ps->d_train_bitmap, n_words, st);
  ps->have_train_norm = false;
  int32_t* d_err = ps->h[0].err;
  CK(cudaMemsetAsync(d_err, 0, sizeof(int32_t), st));
  if (precompute) {
    int rc = launch_pull_norms(c->gdev(), ps->d_train, (int32_t)n_train, ps->d_train_bitmap,
                               ps->d_train_norm, d_err, st);
    if (rc) return rc;
    ps->have_train_norm = true;
  }
  // per-worker local candidate lists (local mode, training.py:236-242)
  std::vector<int32_t> owner(c->n);
  CK(cudaMemcpy(owner.data(), c->d_owner, sizeof(int32_t) * c->n, cudaMemcpyDeviceToHost));
  std::vector<std::vector<int32_t>> loc(c->n_workers);
  for (int64_t i = 0; i < n_train; ++i) loc[owner[t32[i]]].push_back(t32[i]);
  for (int w = 0; w < c->n_workers; ++w) {
    ps->n_local[w] = (int64_t)loc[w].size();
    if (loc[w].empty()) continue;
    CK(cudaMalloc(&ps->d_local[w], sizeof(int32_t) * loc[w].size()));
    CK(cudaMalloc(&ps->d_local_norm[w], sizeof(double) * loc[w].size()));
    CK(cudaMemcpy(ps->d_local[w], loc[w].data(), sizeof(int32_t) * loc[w].size(), cudaMemcpyHostToDevice));
  }
  CK(cudaStreamSynchronize(st));
  int err = 0;
  CK(cudaMemcpy(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
  return status_from_err(err);
}

static int saint_sample(skg_plans* ps, int n, const int32_t* workers, int mode, double D,
                        double min_scale, const skg_rng* rngs, const uint64_t* rng, void* stream) {
  ARG(ps && ps->kind == KIND_SAINT, "not a SAINT plan set");
  ARG(ps->d_train, "call skg_saint_set_candidates first");
  ARG(n >= 1 && n <= ps->n_slots, "slot count out of range");
  skg_ctx* c = ps->ctx;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  {
    const int urc = staging_ready(ps);  // the pinned staging (uniforms) is free again
    if (urc) return urc;
  }
  CK(cudaMemsetAsync(ps->d_scal, 0, ps->scal_bytes, st));
  for (int i = 0; i < n; ++i) {
    const int w = workers[i];
    ARG(w >= 0 && w < c->n_workers, "worker id out of range");
    PlanDev& P = ps->h[i];
    P.worker = w;
    P.mode = mode;
    P.D = D;
    P.min_scale = min_scale;
    int rc = set_rng(ps, P, i, rngs, rng);
    if (rc) return rc;
    if (mode == MODE_LOCAL) {
      if (ps->n_local[w] == 0) {
        set_error("no local training nodes to sample a subgraph from");
        return SKG_ERR_ARG;
      }
      if (!ps->local_norm_ready[w]) {  // column_norms(g, train, local) (training.py:243-244)
        int rc = launch_pull_norms(c->gdev(), ps->d_local[w], (int32_t)ps->n_local[w],
                                   ps->d_train_bitmap, ps->d_local_norm[w], P.err, st);
        if (rc) return rc;
        ps->local_norm_ready[w] = true;
      }
      P.batch = ps->d_local[w];
      P.batch_len = (int32_t)ps->n_local[w];
      P.cand_norm = ps->d_local_norm[w];
      P.budget = std::min<int64_t>(ps->budget, ps->n_local[w]);
    } else {
      if (!ps->have_train_norm) {
        int rc = launch_pull_norms(c->gdev(), ps->d_train, (int32_t)ps->n_train, ps->d_train_bitmap,
                                   ps->d_train_norm, P.err, st);
        if (rc) return rc;
        ps->have_train_norm = true;
      }
      P.batch = ps->d_train;
      P.batch_len = (int32_t)ps->n_train;
      P.cand_norm = ps->d_train_norm;
      P.budget = std::min<int64_t>(ps->budget, ps->n_train);
    }
  }
  {
    const int prc = upload_plans(ps, n, 0, st);
    if (prc) return prc;
  }
  return launch_saint(c->gdev(), ps->d_plans, n, ps->cap_rows, ps->cap_cand, ps->cap_pairs,
                      (int)ps->budget, st);
}

extern "C" int skg_saint_sample(skg_plans* ps, int n, const int32_t* workers, int mode, double D,
                                double min_scale, const uint64_t* rng, void* stream) {
  ARG(rng, "bad arguments");
  return saint_sample(ps, n, workers, mode, D, min_scale, nullptr, rng, stream);
}

extern "C" int skg_saint_sample_rng(skg_plans* ps, int n, const int32_t* workers, int mode, double D,
                                    double min_scale, const skg_rng* rngs, void* stream) {
  ARG(rngs, "bad arguments");
  return saint_sample(ps, n, workers, mode, D, min_scale, rngs, nullptr, stream);
}

__global__ void k_ledger_add(const PlanDev* plans, int L, int64_t* ledger, int32_t* sticky) {
  SKG_PDL_PROLOGUE();
  const PlanDev& P = plans[blockIdx.x];
  if (threadIdx.x == 0 && *P.err) atomicOr(sticky, *P.err);
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    // reference layer order is bottom-up: layer l <-> top-down t = L-1-l (LADIES);
    // SAINT charges its remote count at layer 0 only (training.py:248-253)
    int v, l;
    if (P.kind == KIND_LADIES) {
      v = P.stat[t].remote;
      l = L - 1 - t;
    } else {
      v = t == 0 ? P.stat[0].remote : 0;
      l = t;
    }
    ledger[(int64_t)P.worker * L + l] += v;
  }
}

extern "C" int skg_plans_ledger_add(skg_plans* ps, int slot0, int n, uint64_t ledger_dev,
                                    void* stream) {
  ARG(ps && slot0 >= 0 && n >= 1 && slot0 + n <= ps->n_slots && ledger_dev, "bad ledger arguments");
  cudaStream_t st = (cudaStream_t)stream;
  launch_k("k_ledger_add", st, dim3(n), dim3(32), 0, k_ledger_add, ps->d_plans + slot0, ps->L, (int64_t*)ledger_dev,
           ps->d_sticky);
  CK(cudaGetLastError());
  return SKG_OK;
}

// errors of every plan consumed since the last clear (sampling errors and the training
// step's "no labeled nodes"), which later sampling calls into the arena cannot erase
extern "C" int skg_plans_sticky_error(skg_plans* ps, int clear) {
  ARG(ps, "null plan set");
  CK(cudaSetDevice(ps->ctx->device));
  CK(cudaDeviceSynchronize());
  int32_t err = 0;
  CK(cudaMemcpy(&err, ps->d_sticky, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (clear) CK(cudaMemset(ps->d_sticky, 0, sizeof(int32_t)));
  return status_from_err(err);
}

extern "C" int skg_plan_stats(skg_plans* ps, int slot, int64_t* stats, int64_t info[4]) {
  ARG(ps && slot >= 0 && slot < ps->n_slots, "slot out of range");
  CK(cudaSetDevice(ps->ctx->device));
  CK(cudaDeviceSynchronize());
  const PlanDev& P = ps->h[slot];
  std::vector<LayerStat> ls(ps->L);
  CK(cudaMemcpy(ls.data(), P.stat, sizeof(LayerStat) * ps->L, cudaMemcpyDeviceToHost));
  int32_t err = 0;
  int64_t draws = 0;
  CK(cudaMemcpy(&err, P.err, sizeof(int32_t), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&draws, P.draws_consumed, sizeof(int64_t), cudaMemcpyDeviceToHost));
  int64_t starv = 0;
  const int Ls = ps->kind == KIND_LADIES ? ps->L : 1;
  for (int t = 0; t < Ls; ++t) {
    const LayerStat& s = ls[t];
    int64_t* o = stats + 16 * t;
    o[0] = s.n_upper;
    o[1] = s.n_cand;
    o[2] = s.n_nodes;
    o[3] = s.nnz;
    o[4] = s.remote;
    o[5] = s.has_dist;
    o[6] = s.n_remote_cand;
    o[7] = s.starved;
    o[8] = s.skew;
    o[9] = s.n_pairs;
    o[10] = s.kept_pairs;
    memcpy(&o[11], &s.s, 8);
    memcpy(&o[12], &s.total, 8);
    memcpy(&o[13], &s.T, 8);
    o[14] = s.pw_depth;
    o[15] = 0;
    starv += s.starved;
  }
  info[0] = err;
  info[1] = draws;
  info[2] = starv;
  info[3] = ps->L;
  return status_from_err(err);
}

extern "C" int skg_plan_layer(skg_plans* ps, int slot, int t, int32_t* nodes, int32_t* indptr,
                              int32_t* indices, double* values, int32_t* cand, double* norm,
                              uint8_t* is_local) {
  ARG(ps && slot >= 0 && slot < ps->n_slots, "slot out of range");
  ARG(t >= 0 && t < ps->L, "layer out of range");
  CK(cudaSetDevice(ps->ctx->device));
  CK(cudaDeviceSynchronize());
  const PlanDev& P = ps->h[slot];
  const int ts = ps->kind == KIND_LADIES ? t : 0;
  LayerStat s;
  CK(cudaMemcpy(&s, P.stat + ts, sizeof(LayerStat), cudaMemcpyDeviceToHost));
  if (nodes && s.n_nodes)
    CK(cudaMemcpy(nodes, P.nodes + (size_t)ts * P.cap_rows, 4 * (size_t)s.n_nodes, cudaMemcpyDeviceToHost));
  if (indptr)
    CK(cudaMemcpy(indptr, P.indptr + (size_t)ts * (P.cap_rows + 1), 4 * (size_t)(s.n_upper + 1), cudaMemcpyDeviceToHost));
  if (indices && s.nnz)
    CK(cudaMemcpy(indices, P.indices + (size_t)ts * P.cap_pairs, 4 * (size_t)s.nnz, cudaMemcpyDeviceToHost));
  if (values && s.nnz)
    CK(cudaMemcpy(values, P.val + (size_t)ts * P.cap_pairs, 8 * (size_t)s.nnz, cudaMemcpyDeviceToHost));
  if (s.n_cand) {
    const int32_t* cp;
    const double* np_;
    if (ps->kind == KIND_SAINT) {
      cp = P.batch;
      np_ = P.cand_norm ? P.cand_norm : P.norm;
    } else {
      cp = P.cand + (size_t)ts * P.cap_cand;
      np_ = P.norm + (size_t)ts * P.cap_cand;
    }
    if (cand) CK(cudaMemcpy(cand, cp, 4 * (size_t)s.n_cand, cudaMemcpyDeviceToHost));
    if (norm) CK(cudaMemcpy(norm, np_, 8 * (size_t)s.n_cand, cudaMemcpyDeviceToHost));
    if (is_local)
      CK(cudaMemcpy(is_local, P.is_local + (size_t)ts * P.cap_cand, (size_t)s.n_cand, cudaMemcpyDeviceToHost));
  }
  return SKG_OK;
}

// ------------------------------------------------------------------ GCN
extern "C" int skg_gcn_create(skg_plans* ps, int L, const int64_t* dims, int dtype, skg_gcn** out) {
  ARG(ps && out && dims && L == ps->L, "GCN depth must match the plan depth");
  ARG(dtype == DT_F32 || dtype == DT_F64, "bad dtype");
  ARG(ps->ctx->d_x && ps->ctx->F == dims[0], "features missing or dim mismatch");
  ARG(ps->ctx->dtype == dtype, "feature dtype must equal the compute dtype");
  CK(cudaSetDevice(ps->ctx->device));
  skg_gcn* g = new skg_gcn();
  g->ps = ps;
  g->L = L;
  g->dtype = dtype;
  g->n_slots = ps->n_slots;
  g->dims.assign(dims, dims + L + 1);
  g->ld.resize(L + 1);
  int64_t wmax = 0;
  for (int l = 0; l <= L; ++l) {
    g->ld[l] = round4(dims[l]);
    g->ld_max = std::max(g->ld_max, g->ld[l]);
    if (l < L) wmax = std::max(wmax, dims[l] * dims[l + 1]);
  }
  const size_t es = dtype == DT_F32 ? 4 : 8;
  const int64_t R = ps->cap_rows, S = ps->n_slots;
  g->R = R;
  g->part_elems = wmax;
  g->U.resize(L);
  g->H.resize(L + 1);
  Carver cv;
  for (int l = 0; l < L; ++l) cv.add(g->U[l], (size_t)S * R * g->ld[l] * es);
  for (int l = 1; l <= L; ++l) cv.add(g->H[l], (size_t)S * R * g->ld[l] * es);
  cv.add(g->G0, (size_t)S * R * g->ld_max * es);
  cv.add(g->G1, (size_t)S * R * g->ld_max * es);
  cv.add(g->G2, (size_t)S * R * g->ld_max * es);
  if (dtype == DT_F32) {
    g->Ulo.resize(L);
    g->Wh.resize(L);
    g->Wl.resize(L);
    g->ldw.resize(L);
    for (int l = 0; l < L; ++l) {
      cv.add(g->Ulo[l], (size_t)S * R * g->ld[l] * es);
      g->ldw[l] = round4(dims[l + 1]);
      cv.add(g->Wh[l], (size_t)dims[l] * g->ldw[l] * es);
      cv.add(g->Wl[l], (size_t)dims[l] * g->ldw[l] * es);
    }
    cv.add(g->G0lo, (size_t)S * R * g->ld_max * es);
    cv.add(g->G2lo, (size_t)S * R * g->ld_max * es);
  }
  cv.add(g->parts, (size_t)S * kMaxKSplit * wmax * es);
  cv.add(g->row_loss, (size_t)S * R);
  cv.add(g->nlab, (size_t)S);
  cv.add(g->d_layers, (size_t)L * S);
  cv.add(g->d_slots, (size_t)S);
  cv.add(g->d_rows, (size_t)L * S);
  CK(cudaMalloc(&g->arena, cv.off));
  CK(cudaMemset(g->arena, 0, cv.off));
  cv.bind(g->arena);
  CK(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
  g->ev.resize(2 * L + 4);
  for (auto& e : g->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // descriptors: pointers into the plan arena are fixed for the plan set's lifetime
  std::vector<LayerDesc> hl((size_t)L * S);
  std::vector<const int32_t*> hr((size_t)L * S);
  std::vector<SlotDesc> hs(S);
  for (int z = 0; z < S; ++z) {
    const PlanDev& P = ps->h[z];
    for (int l = 0; l < L; ++l) {
      const int t = ps->kind == KIND_LADIES ? L - 1 - l : 0;
      LayerDesc d;
      d.rows = &P.stat[t].n_upper;
      d.cols = &P.stat[t].n_nodes;
      d.indptr = P.indptr + (size_t)t * (P.cap_rows + 1);
      d.indices = P.indices + (size_t)t * P.cap_pairs;
      d.val = P.val + (size_t)t * P.cap_pairs;
      d.tindptr = P.tindptr + (size_t)t * (P.cap_rows + 1);
      d.tindices = P.tindices + (size_t)t * P.cap_pairs;
      d.tval = P.tval + (size_t)t * P.cap_pairs;
      hl[(size_t)l * S + z] = d;
      hr[(size_t)l * S + z] = d.rows;
    }
    const int t0 = ps->kind == KIND_LADIES ? L - 1 : 0;
    SlotDesc sd;
    sd.in_nodes = P.nodes + (size_t)t0 * P.cap_rows;
    sd.n_in = &P.stat[t0].n_nodes;
    sd.batch = ps->kind == KIND_LADIES ? nullptr : P.nodes;  // LADIES: set per sampling call
    sd.n_batch = ps->kind == KIND_LADIES ? &P.stat[0].n_upper : &P.stat[0].n_nodes;
    sd.err = P.err;
    hs[z] = sd;
  }
  CK(cudaMemcpy(g->d_layers, hl.data(), sizeof(LayerDesc) * hl.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(g->d_rows, hr.data(), sizeof(void*) * hr.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(g->d_slots, hs.data(), sizeof(SlotDesc) * hs.size(), cudaMemcpyHostToDevice));
  *out = g;
  return SKG_OK;
}

// loss of the GCN head: 0 softmax cross-entropy, 1 multi-label BCE-with-logits with
// positive-class weight pos_weight (mean over rows x classes)
extern "C" int skg_gcn_set_loss(skg_gcn* g, int kind, double pos_weight) {
  ARG(g && (kind == 0 || kind == 1) && pos_weight > 0.0, "bad loss");
  g->loss_kind = kind;
  g->pos_weight = pos_weight;
  return SKG_OK;
}

extern "C" int skg_gcn_destroy(skg_gcn* g) {
  if (!g) return SKG_OK;
  g->graphs.clear();
  for (cudaEvent_t e : g->ev) cudaEventDestroy(e);
  if (g->side) cudaStreamDestroy(g->side);
  if (g->graphs.cap) cudaStreamDestroy(g->graphs.cap);
  if (g->loss_scratch) cudaFree(g->loss_scratch);
  cudaFree(g->arena);
  delete g;
  return SKG_OK;
}

namespace {
// LADIES batch pointers change with every sampling call (they point at the caller's
// batch buffer); refresh them in the slot descriptors before running.
int refresh_batches(skg_gcn* g, int z0, int n, cudaStream_t st) {
  skg_plans* ps = g->ps;
  if (ps->kind != KIND_LADIES) return SKG_OK;
  if ((int)g->batch_seen.size() != g->n_slots) g->batch_seen.assign(g->n_slots, nullptr);
  for (int z = z0; z < z0 + n; ++z) {
    const int32_t* b = ps->h[z].batch;
    if (b == g->batch_seen[z]) continue;  // unchanged since the last write
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(g->d_slots + z) + offsetof(SlotDesc, batch), &b,
                       sizeof(b), cudaMemcpyHostToDevice, st));
    g->batch_seen[z] = b;
  }
  return SKG_OK;
}

template <typename T>
Act<T> act(char* base, int64_t R, int64_t ld_alloc, int64_t ld, int z0, size_t es = sizeof(T)) {
  Act<T> a;
  a.base = reinterpret_cast<T*>(base) + (int64_t)z0 * R * ld_alloc;
  a.stride = R * ld_alloc;
  a.ld = ld;
  return a;
}

template <typename T>
int gcn_run(skg_gcn* g, int z0, int n, const uint64_t* wp, const uint64_t* gp, bool accum,
            double* loss, bool backward, cudaStream_t st) {
  skg_plans* ps = g->ps;
  skg_ctx* c = ps->ctx;
  const int L = g->L, S = g->n_slots;
  const int64_t R = g->R;
  const int Ri = (int)R;
  int rc = SKG_OK;
  // fp32 GEMMs on tcgen05 (mode 1 / 3) read TF32-split operands; 3xTF32 also needs lo parts
  constexpr bool F32 = sizeof(T) == 4;
  const int mode = F32 ? g_gemm_mode : 0;
  const bool tc = mode != 0, split = mode == 3;
  auto W = [&](int l) {
    Act<T> a;
    a.base = reinterpret_cast<T*>(wp[l]);
    a.stride = 0;
    a.ld = g->dims[l + 1];
    return a;
  };
  auto lo_of = [&](char* base, int64_t ld_alloc) -> T* {
    return split ? reinterpret_cast<T*>(base) + (int64_t)z0 * R * ld_alloc : nullptr;
  };
  auto op = [&](char* hi, char* lo, int64_t ld_alloc, int64_t ld) {
    TcOp o;
    o.hi = reinterpret_cast<const float*>(hi) + (int64_t)z0 * R * ld_alloc;
    o.lo = split ? reinterpret_cast<const float*>(lo) + (int64_t)z0 * R * ld_alloc : nullptr;
    o.ld = ld;
    o.stride = R * ld_alloc;
    o.rows_cap = R;
    return o;
  };
  auto wop = [&](int l) {
    TcOp o;
    o.hi = reinterpret_cast<const float*>(g->Wh[l]);
    o.lo = split ? reinterpret_cast<const float*>(g->Wl[l]) : nullptr;
    o.ld = g->ldw[l];
    o.stride = 0;
    o.rows_cap = g->dims[l];
    return o;
  };
  // side branch at the start: the TF32 weight split (needed by the first GEMM) and the
  // labelled-row count (needed by the softmax) run beside the gather and the first SpMM
  cudaStream_t sd = g->side;
  const bool soft = backward && g->loss_kind == 0;
  CK(cudaEventRecord(g->ev[2 * L + 1], st));
  CK(cudaStreamWaitEvent(sd, g->ev[2 * L + 1], 0));
  if (soft) count_labels_b(g->d_slots + z0, n, c->d_labels, g->nlab + z0, sd);
  if (tc) {
    WSplitTable t;
    t.L = L;
    for (int l = 0; l < L; ++l) {
      t.w[l] = reinterpret_cast<const float*>(wp[l]);
      t.hi[l] = reinterpret_cast<float*>(g->Wh[l]);
      t.lo[l] = split ? reinterpret_cast<float*>(g->Wl[l]) : nullptr;
      t.rows[l] = g->dims[l];
      t.cols[l] = g->dims[l + 1];
      t.ld_out[l] = g->ldw[l];
    }
    split_weights(t, sd);
  }
  CK(cudaEventRecord(g->ev[2 * L + 2], sd));
  for (int l = 0; l < L; ++l) {
    const LayerDesc* lds = g->d_layers + (size_t)l * S + z0;
    const int32_t* const* rows = g->d_rows + (size_t)l * S + z0;
    Act<T> U = act<T>(g->U[l], R, g->ld[l], g->ld[l], z0);
    if (l == 0) {  // the X[S_0] gather (local or NVLink peer rows) fused into the first SpMM
      spmm_in_b<T>(c->fstore(), g->d_slots + z0, lds, n, Ri, U, F32 ? lo_of(g->Ulo[0], g->ld[0]) : nullptr,
                   g->ld[0], st);
    } else {
      Act<T> A = act<T>(g->H[l], R, g->ld[l], g->ld[l], z0);
      spmm_b<T>(lds, n, Ri, false, true, A, A, U, F32 ? lo_of(g->Ulo[l], g->ld[l]) : nullptr, g->ld[l], st);
    }
    if (l == 0) CK(cudaStreamWaitEvent(st, g->ev[2 * L + 2], 0));  // split weights, label counts
    Act<T> Hn = act<T>(g->H[l + 1], R, g->ld[l + 1], g->ld[l + 1], z0);
    if constexpr (F32) {
      if (tc) {
        g_gemm_layer = l;
        rc = gemm_tc(mode, false, false, n, Ri, (int)g->dims[l + 1], (int)g->dims[l], rows, nullptr,
                     op(g->U[l], g->Ulo[l], g->ld[l], g->ld[l]), wop(l), Hn, false, st);
        if (rc) return rc;
        continue;
      }
    }
    gemm_simt<T>(false, false, n, Ri, (int)g->dims[l + 1], (int)g->dims[l], rows, nullptr, U, W(l), Hn,
                 false, st);
  }
  g_gemm_layer = -1;
  if (!backward) return SKG_OK;
  // G alternates between G0 and G2: the dW GEMM of layer l (on the side stream) reads the
  // buffer the transposed SpMM of layer l - 1 would otherwise overwrite
  char* Gb[2] = {g->G0, g->G2};
  char* Gl[2] = {g->G0lo, g->G2lo};
  int cur = 0;
  Act<T> G = act<T>(Gb[0], R, g->ld_max, g->ld[L], z0);
  Act<T> Gu = act<T>(g->G1, R, g->ld_max, g->ld[L], z0);
  T* G_lo = F32 ? lo_of(Gl[0], g->ld_max) : nullptr;
  if (g->loss_kind == 1) {
    if (!c->d_ymulti || c->y_classes != g->dims[L]) {
      set_error("multi-label BCE needs multi-hot labels with one bit per output class");
      return SKG_ERR_ARG;
    }
    bce_b<T>(g->d_slots + z0, n, Ri, c->d_ymulti, c->y_words, act<T>(g->H[L], R, g->ld[L], g->ld[L], z0),
             (int)g->dims[L], g->pos_weight, G, G_lo, g->row_loss + (size_t)z0 * R, loss, st);
  } else {
    softmax_ce_rows_b<T>(g->d_slots + z0, n, Ri, c->d_labels, act<T>(g->H[L], R, g->ld[L], g->ld[L], z0),
                         (int)g->dims[L], G, G_lo, g->row_loss + (size_t)z0 * R, g->nlab + z0, st);
    // the fixed-order loss mean runs beside the backward chain
    CK(cudaEventRecord(g->ev[2 * L + 3], st));
    CK(cudaStreamWaitEvent(sd, g->ev[2 * L + 3], 0));
    loss_mean_b(g->d_slots + z0, n, Ri, c->d_labels, g->row_loss + (size_t)z0 * R, g->nlab + z0, loss, sd);
  }
  for (int l = L - 1; l >= 0; --l) {
    const LayerDesc* lds = g->d_layers + (size_t)l * S + z0;
    const int32_t* const* rows = g->d_rows + (size_t)l * S + z0;
    const int dl = (int)g->dims[l], dn = (int)g->dims[l + 1];
    // dW_l = sum_slots U_l^T G (split-K over slots, reduced in slot order), on the side
    // stream: nothing on the dX -> SpMM^T chain waits for it
    CK(cudaEventRecord(g->ev[l], st));
    CK(cudaStreamWaitEvent(sd, g->ev[l], 0));
    Act<T> P;
    P.base = reinterpret_cast<T*>(g->parts);
    P.stride = g->part_elems;
    P.ld = dn;
    bool done = false;
    int ks = 1;  // K split inside each slot: partial (slot, run) blocks in slot-major order
    if constexpr (F32) {
      if (tc) {
        g_gemm_layer = l;
        ks = gemm_tc_ksplit(n, dl, dn, Ri);
        rc = gemm_tc(mode, true, false, n, dl, dn, Ri, nullptr, rows, op(g->U[l], g->Ulo[l], g->ld[l], g->ld[l]),
                     op(Gb[cur], Gl[cur], g->ld_max, G.ld), P, false, sd, ks);
        if (rc) return rc;
        done = true;
      }
    }
    if (!done)
      gemm_simt<T>(true, false, n, dl, dn, Ri, nullptr, rows, act<T>(g->U[l], R, g->ld[l], g->ld[l], z0), G,
                   P, false, sd);
    reduce_slots<T>(P.base, P.stride, n * ks, dl, dn, dn, reinterpret_cast<T*>(gp[l]), dn, accum, sd);
    CK(cudaEventRecord(g->ev[L + l], sd));
    if (l == 0) break;
    // G_u = G W_l^T ; G <- (Block_l^T G_u) * [H_l > 0]
    Gu.ld = g->ld[l];
    done = false;
    if constexpr (F32) {
      if (tc) {
        g_gemm_layer = l;
        rc = gemm_tc(mode, false, true, n, Ri, dl, dn, rows, nullptr, op(Gb[cur], Gl[cur], g->ld_max, G.ld), wop(l),
                     Gu, false, st);
        if (rc) return rc;
        done = true;
      }
    }
    if (!done) gemm_simt<T>(false, true, n, Ri, dl, dn, rows, nullptr, G, W(l), Gu, false, st);
    // the other G buffer was read by dW_{l+1}
    if (l + 1 < L) CK(cudaStreamWaitEvent(st, g->ev[L + l + 1], 0));
    Act<T> Gn = act<T>(Gb[cur ^ 1], R, g->ld_max, g->ld[l], z0);
    spmm_b<T>(lds, n, Ri, true, false, Gu, act<T>(g->H[l], R, g->ld[l], g->ld[l], z0), Gn,
              F32 ? lo_of(Gl[cur ^ 1], g->ld_max) : nullptr, g->ld[l], st);
    G = Gn;
    cur ^= 1;
  }
  CK(cudaEventRecord(g->ev[2 * L], sd));  // join: the step ends when every dW is reduced
  CK(cudaStreamWaitEvent(st, g->ev[2 * L], 0));
  g_gemm_layer = -1;
  return SKG_OK;
}

int gcn_eager(skg_gcn* g, int z0, int n, const uint64_t* wp, const uint64_t* gp, bool acc,
              double* loss, bool backward, cudaStream_t st) {
  return g->dtype == DT_F32 ? gcn_run<float>(g, z0, n, wp, gp, acc, loss, backward, st)
                            : gcn_run<double>(g, z0, n, wp, gp, acc, loss, backward, st);
}

// Everything a captured step bakes into its launches: slots, weight / gradient buffers,
// flags, loss head, GEMM configuration and the context's data pointers (generation).
std::string graph_key(const skg_gcn* g, int z0, int n, const uint64_t* wp, const uint64_t* gp, bool acc) {
  std::string k;
  auto put = [&](const void* p, size_t b) { k.append(reinterpret_cast<const char*>(p), b); };
  const int hdr[7] = {z0, n, acc ? 1 : 0, g->loss_kind, g_gemm_mode, g_bn_override, g_ksplit_override};
  put(hdr, sizeof(hdr));
  put(&g->pos_weight, sizeof(double));
  put(&g->ps->ctx->gen, sizeof(uint64_t));
  put(wp, sizeof(uint64_t) * g->L);
  put(gp, sizeof(uint64_t) * g->L);
  return k;
}

int gcn_dispatch(skg_gcn* g, int z0, int n, const uint64_t* wp, const uint64_t* gp, bool acc,
                 double* loss, bool backward, cudaStream_t st, bool repeat = false) {
  int rc = refresh_batches(g, z0, n, st);
  if (rc) return rc;
  if (backward && loss && gp && graphs_on()) {
    // training step: replay a CUDA graph of its ~45 launches
    if (!g->loss_scratch) CK(cudaMalloc(&g->loss_scratch, sizeof(double) * std::max(g->n_slots, 1)));
    rc = graph_run(g->graphs, graph_key(g, z0, n, wp, gp, acc), st, repeat, [&](cudaStream_t cs) {
      return gcn_eager(g, z0, n, wp, gp, acc, g->loss_scratch, true, cs);
    });
    if (rc) return rc;
    CK(cudaMemcpyAsync(loss, g->loss_scratch, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  } else {
    rc = gcn_eager(g, z0, n, wp, gp, acc, loss, backward, st);
    if (rc) return rc;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("gcn: ") + cudaGetErrorString(e));
    return SKG_ERR_CUDA;
  }
  return SKG_OK;
}
}  // namespace

extern "C" int skg_gcn_step(skg_gcn* g, int slot, const uint64_t* wp, const uint64_t* gp,
                            int accumulate, uint64_t loss_dev, void* stream) {
  ARG(g && slot >= 0 && slot < g->n_slots && wp && gp && loss_dev, "bad gcn_step arguments");
  ARG(g->ps->ctx->d_labels || g->ps->ctx->d_ymulti, "labels not set");
  CK(cudaSetDevice(g->ps->ctx->device));
  return gcn_dispatch(g, slot, 1, wp, gp, accumulate != 0, (double*)loss_dev, true,
                      (cudaStream_t)stream);
}

extern "C" int skg_gcn_step_batch(skg_gcn* g, int slot0, int n, const uint64_t* wp,
                                  const uint64_t* gp, int accumulate, uint64_t loss_dev,
                                  void* stream) {
  ARG(g && slot0 >= 0 && n >= 1 && slot0 + n <= g->n_slots && wp && gp && loss_dev,
      "bad gcn_step_batch arguments");
  ARG(g->ps->ctx->d_labels || g->ps->ctx->d_ymulti, "labels not set");
  CK(cudaSetDevice(g->ps->ctx->device));
  // the batched step is the Trainer's: its keys repeat every group
  return gcn_dispatch(g, slot0, n, wp, gp, accumulate != 0, (double*)loss_dev, true,
                      (cudaStream_t)stream, true);
}

extern "C" int skg_gcn_forward(skg_gcn* g, int slot, const uint64_t* wp, void* stream) {
  ARG(g && slot >= 0 && slot < g->n_slots && wp, "bad gcn_forward arguments");
  CK(cudaSetDevice(g->ps->ctx->device));
  return gcn_dispatch(g, slot, 1, wp, nullptr, false, nullptr, false, (cudaStream_t)stream);
}

extern "C" int skg_gcn_read_logits(skg_gcn* g, int slot, void* host_out, int64_t* rows_out) {
  ARG(g && slot >= 0 && slot < g->n_slots, "bad slot");
  CK(cudaSetDevice(g->ps->ctx->device));
  CK(cudaDeviceSynchronize());
  skg_plans* ps = g->ps;
  const PlanDev& P = ps->h[slot];
  LayerStat s;
  CK(cudaMemcpy(&s, P.stat + 0, sizeof(LayerStat), cudaMemcpyDeviceToHost));
  const int64_t rows = s.n_upper;
  *rows_out = rows;
  const size_t es = g->dtype == DT_F32 ? 4 : 8;
  const int64_t C = g->dims[g->L];
  const char* src = g->H[g->L] + (size_t)slot * g->R * g->ld[g->L] * es;
  if (host_out && rows)
    CK(cudaMemcpy2D(host_out, es * C, src, es * g->ld[g->L], es * C, rows, cudaMemcpyDeviceToHost));
  return SKG_OK;
}

extern "C" int skg_predict_logits(skg_ctx* c, int L, const int64_t* dims, const uint64_t* wp,
                                  int dtype, uint64_t out_dev, void* stream) {
  ARG(c && dims && wp && out_dev && L >= 1, "bad predict arguments");
  ARG(c->d_x && c->dtype == dtype && c->F == dims[0] && c->x_rows == c->n,
      "full-graph inference needs all feature rows on this device");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t es = dtype == DT_F32 ? 4 : 8;
  int64_t ldm = 0;
  for (int l = 0; l <= L; ++l) ldm = std::max(ldm, round4(dims[l]));
  char *U = nullptr, *H = nullptr, *Ul = nullptr, *Wh = nullptr, *Wl = nullptr;
  const int mode = dtype == DT_F32 ? g_gemm_mode : 0;  // fp32: tcgen05 on TF32-split operands
  int64_t wmax = 0;
  for (int l = 0; l < L; ++l) wmax = std::max(wmax, dims[l] * round4(dims[l + 1]));
  CK(cudaMalloc(&U, es * ldm * std::max<int64_t>(c->n, 1)));
  CK(cudaMalloc(&H, es * ldm * std::max<int64_t>(c->n, 1)));
  CK(cudaMemsetAsync(H, 0, es * ldm * std::max<int64_t>(c->n, 1), st));
  if (mode) {
    CK(cudaMalloc(&Ul, es * ldm * std::max<int64_t>(c->n, 1)));
    CK(cudaMalloc(&Wh, es * std::max<int64_t>(wmax, 1)));
    CK(cudaMalloc(&Wl, es * std::max<int64_t>(wmax, 1)));
  }
  int rc = SKG_OK;
  for (int l = 0; l < L; ++l) {
    const int64_t ldi = l == 0 ? c->ldx : round4(dims[l]);
    const int64_t ldl = round4(dims[l]);
    const bool last = l == L - 1;
    const int64_t ldo = last ? dims[L] : round4(dims[l + 1]);
    if (dtype == DT_F32) {
      const float* A = l == 0 ? (const float*)c->d_x : (const float*)H;
      if (l == 0 && c->xbits)
        spmm_full_bits<float>(c->n, c->d_off, c->d_col, c->d_w, (const uint32_t*)c->d_x, c->ldx, (float*)U, ldl,
                              ldl, st);
      else
        spmm_full<float>(c->n, c->d_off, c->d_col, c->d_w, A, ldi, l > 0, (float*)U, ldl, ldl, st);
      if (mode) {
        // P·(X·W) rounding differs from the fp64 reference only at fp32 level (3xTF32)
        float* uh = (float*)U;
        float* ul = mode == 3 ? (float*)Ul : nullptr;
        split_tf32(uh, ldl, c->n, dims[l], uh, ul, ldl, st);  // in place: hi over U
        const int64_t ldw = round4(dims[l + 1]);
        split_tf32((const float*)wp[l], dims[l + 1], dims[l], dims[l + 1], (float*)Wh,
                   mode == 3 ? (float*)Wl : nullptr, ldw, st);
        TcOp a{uh, ul, ldl, 0, c->n}, b{(const float*)Wh, mode == 3 ? (const float*)Wl : nullptr, ldw, 0, dims[l]};
        Act<float> out{last ? (float*)out_dev : (float*)H, 0, ldo};
        rc = gemm_tc(mode, false, false, 1, (int)c->n, (int)dims[l + 1], (int)dims[l], nullptr, nullptr, a, b,
                     out, false, st);
        if (rc) break;
      } else {
        gemm_plain<float>((int)c->n, (int)dims[l + 1], (int)dims[l], (const float*)U, ldl,
                          (const float*)wp[l], dims[l + 1], last ? (float*)out_dev : (float*)H, ldo, st);
      }
    } else {
      const double* A = l == 0 ? (const double*)c->d_x : (const double*)H;
      if (l == 0 && c->xbits)
        spmm_full_bits<double>(c->n, c->d_off, c->d_col, c->d_w, (const uint32_t*)c->d_x, c->ldx, (double*)U,
                               ldl, ldl, st);
      else
        spmm_full<double>(c->n, c->d_off, c->d_col, c->d_w, A, ldi, l > 0, (double*)U, ldl, ldl, st);
      gemm_plain<double>((int)c->n, (int)dims[l + 1], (int)dims[l], (const double*)U, ldl,
                         (const double*)wp[l], dims[l + 1], last ? (double*)out_dev : (double*)H, ldo,
                         st);
    }
  }
  cudaStreamSynchronize(st);
  cudaFree(U);
  cudaFree(H);
  if (Ul) cudaFree(Ul);
  if (Wh) cudaFree(Wh);
  if (Wl) cudaFree(Wl);
  if (rc) return rc;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("predict_logits: ") + cudaGetErrorString(e));
    return SKG_ERR_CUDA;
  }
  return SKG_OK;
}

extern "C" int skg_sgd_step(int dtype, uint64_t w, uint64_t g, int64_t n, double lr, double contrib,
                            void* stream) {
  ARG(n >= 0 && contrib > 0, "bad sgd arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == DT_F32) sgd_step<float>((float*)w, (const float*)g, n, lr, contrib, st);
  else sgd_step<double>((double*)w, (const double*)g, n, lr, contrib, st);
  CK(cudaGetLastError());
  return SKG_OK;
}

extern "C" int skg_adam_step(int dtype, uint64_t w, uint64_t g, uint64_t m, uint64_t v, int64_t n,
                             double lr, double contrib, int64_t t, void* stream) {
  ARG(n >= 0 && contrib > 0 && t >= 1, "bad adam arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  const double bc1 = 1.0 - std::pow(b1, (double)t), bc2 = 1.0 - std::pow(b2, (double)t);
  if (dtype == DT_F32)
    adam_step<float>((float*)w, (const float*)g, (float*)m, (float*)v, n, lr, contrib, b1, b2,
                     1.0 - b1, 1.0 - b2, bc1, bc2, eps, st);
  else
    adam_step<double>((double*)w, (const double*)g, (double*)m, (double*)v, n, lr, contrib, b1, b2,
                      1.0 - b1, 1.0 - b2, bc1, bc2, eps, st);
  CK(cudaGetLastError());
  return SKG_OK;
}

namespace skg { extern int g_gemm_mode; }
extern "C" int skg_set_gemm_mode(int mode) {
  ARG(mode == 0 || mode == 1 || mode == 3, "gemm mode must be 0 (SIMT), 1 (TF32) or 3 (3xTF32)");
  skg::g_gemm_mode = mode;
  return SKG_OK;
}

extern "C" int skg_zero(int dtype, uint64_t p, int64_t n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == DT_F32) fill_zero<float>((float*)p, n, st);
  else fill_zero<double>((double*)p, n, st);
  CK(cudaGetLastError());
  return SKG_OK;
}
