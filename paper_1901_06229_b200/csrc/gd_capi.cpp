// C-ABI implementation: context, pocket/params upload, host-side ligand validation and SoA packing,
// batch staging, kernel launch, result fetch. See include/geodock_b200.h for the contract and
// DESIGN.md for the layout. Paths in comments are relative to /root/reference/proj.
//
// Host arithmetic that feeds the device (rotation grid, dihedral table, starting transforms) is
// the reference's own FP64 formulas evaluated with the same libm, so the device sees the same
// bits the reference computes (compiled with -ffp-contract=off, no -march).
#include <algorithm>
#include <array>
#include <chrono>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "gd_host_math.h"
#include "gd_ligand.h"
#include "gd_internal.h"
#include "geodock_b200.h"

using gdk::DevBatch;
using gdk::DevParams;
using gdk::DevPocket;
using gdk::LigMeta;

// executor staging slots: three, so one chunk is always queued on the GPU while the host packs the
// next and unpacks the previous
constexpr int kSlots = 3;

// Host worker pool for the executor's per-chunk validation, packing and unpacking: persistent
// threads (the caller works too), so a chunk's host work does not pay thread start-up on the
// critical path. One pool per context (a context is externally synchronized, so one job runs at a
// time), created at the context's first batch; its width is the host's share of this context:
// GD_HOST_THREADS if set, else the hardware threads divided by max(live contexts of this process,
// LOCAL_WORLD_SIZE) — one context per GPU, whether the GPUs are driven by threads of one process
// (run_screening creates every lane's context before docking) or by one process each (torchrun),
// share the cores instead of oversubscribing them, and a lone context on a multi-GPU node gets
// all of them.
class HostPool {
 public:
  explicit HostPool(unsigned threads) {
    for (unsigned t = 0; t + 1 < threads; ++t) th_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  unsigned threads() const { return unsigned(th_.size()) + 1; }
  void run(size_t n, size_t grain, const std::function<void(size_t)>& f) {
    std::lock_guard<std::mutex> s(submit_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      n_ = n;
      grain_ = grain;
      chunks_ = (n + grain - 1) / grain;
      next_.store(0);
      pending_ = unsigned(th_.size());
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }
  static unsigned default_threads() {
    if (const char* e = std::getenv("GD_HOST_THREADS")) {
      const int v = std::atoi(e);
      if (v > 0) return unsigned(v);
    }
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned share = std::max(1, live_contexts.load());
    if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) share = std::max(share, unsigned(std::max(1, std::atoi(e))));
    return std::max(1u, hw / share);
  }
  // contexts alive in this process (gd_create / gd_destroy): the contexts of one process share the
  // host cores, and the ranks of one node (LOCAL_WORLD_SIZE) share them between processes
  static inline std::atomic<int> live_contexts{0};

 private:
  void work() {
    for (;;) {
      const size_t c = next_.fetch_add(1);
      if (c >= chunks_) return;
      const size_t e = std::min(n_, (c + 1) * grain_);
      for (size_t i = c * grain_; i < e; ++i) (*job_)(i);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      lk.unlock();
      work();
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex submit_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(size_t)>* job_ = nullptr;
  size_t n_ = 0, grain_ = 1, chunks_ = 0;
  std::atomic<size_t> next_{0};
  unsigned pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct gd_ctx {
  int device = 0;
  int n_sms = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int mode = GD_MODE_FAST;

  // pocket
  bool have_pocket = false;
  uint32_t dims[3] = {0, 0, 0};
  double origin[3] = {0, 0, 0};
  double spacing = 1.0;
  double* d_field = nullptr;
  uint4* d_cells = nullptr;
  float* d_field_f = nullptr;  // FP32 field + zero tail (K1b's coarse samples)
  uint32_t f_count = 0;
  float q_eps_f = 0.f;
  float q_eps = 0.f;
  float max_step = 0.f;
  float dz_bias = 3.f;

  // params
  gd_params params{};
  bool have_params = false;
  double4* d_grid = nullptr;
  float4* d_grid_f = nullptr;
  float4* d_frames = nullptr;
  uint32_t* d_frame_tab = nullptr;  // K1a frame schedule: kept frames + twin table (upload_grid_f)
  uint32_t n_kept = 0;
  uint32_t n_twin_frames = 0;
  double4* d_dtab = nullptr;
  float2* d_dtab_f = nullptr;
  uint32_t G = 0;
  std::vector<double> grid_host;  // 4 per entry

  gd_stats last{};
  unsigned long long* d_stats = nullptr;
  int* d_error = nullptr;
  unsigned int* d_counter = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // gd_run: K1a | K1b | K2 boundaries

  // executor staging slots (gd_dock_batch): grow-only pinned host buffers + device arena + stream
  struct Slot {
    void* h_in = nullptr;
    size_t h_in_cap = 0;
    void* h_out = nullptr;
    size_t h_out_cap = 0;
    void* d_arena = nullptr;
    size_t d_cap = 0;
    cudaStream_t stream = nullptr;  // copies of this slot
    cudaEvent_t in = nullptr, mid = nullptr, k = nullptr, done = nullptr;  // H2D | K1a | K2 | D2H done
    cudaEvent_t a0 = nullptr;                                             // before K1a (timing)
  } slot[kSlots];
  // executor compute streams: all chunks' K1a in order on sa, their K1b + K2 on sb (so chunk c+1's
  // alignment overlaps chunk c's sweep, and chunks complete in order)
  cudaStream_t sa = nullptr, sb = nullptr;
  // last gd_dock_batch's device accounting (RunMetrics, pipeline.hpp:43-72): busy span (first K1a
  // start to last K2 end), per-chunk K1a and K1b + K2 event intervals, host time waiting on the GPU
  cudaEvent_t run0 = nullptr, run1 = nullptr;
  double run_times[4] = {0, 0, 0, 0};
  HostPool* pool = nullptr;  // host threads of this context (validation, packing, unpacking)
};

struct Layout {
  uint32_t L = 0, A = 0, Rt = 0, max_n = 1, fast_max_n = 0;
  uint32_t class_max_n[3] = {0, 0, 0};  // per fast-kernel class (n <= 32, <= 64, <= 128)
  size_t n_items = 0;
  std::vector<uint32_t> mask_base, adj_base;
  size_t o_meta, o_atoms, o_start, o_rots, o_dih0, o_masks, o_adj, o_dfs, o_rdfs, o_adjd, host_bytes;
  size_t o_cand, o_ncand, o_rs_score, o_rs_ascore, o_rs_aidx, o_rs_stepk, o_rs_pose, o_rs_es, o_rs_ext, o_slow;
  size_t o_best, o_brs, o_fxyz, o_fdih, o_ctr, o_order, o_ord_scr, o_ord_tmp, ord_tmp_bytes = 0, total;
};

struct gd_batch {
  gd_ctx* ctx = nullptr;
  DevBatch dev{};
  void* arena = nullptr;
  size_t arena_bytes = 0;
  void* topk_scratch = nullptr;
  size_t topk_bytes = 0;
  gd_hit* d_hits = nullptr;
  std::vector<uint32_t> atom_off, rot_off, name_off;
  std::string names;  // ligand names (error messages)
  uint32_t n_restarts = 0, reps = 0, S = 0;
  gd_params params{};
  Layout layout;
};

namespace {

int set_err(gd_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_err(gd_ctx* ctx, cudaError_t e, const char* what) {
  return set_err(ctx, GD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define GD_CUDA(ctx, call)                                \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_err(ctx, e_, #call); \
  } while (0)

HostPool& pool_of(gd_ctx* ctx) {
  if (!ctx->pool) ctx->pool = new HostPool(HostPool::default_threads());
  return *ctx->pool;
}

// f(i) for i < n on the context's host threads, in chunks of `grain` indices (0: about 8 chunks
// per thread)
template <class F>
void parallel_for(gd_ctx* ctx, size_t n, size_t grain, F&& f) {
  HostPool& pool = pool_of(ctx);
  const unsigned hw = pool.threads();
  if (grain == 0) grain = std::max<size_t>(1, n / (8 * size_t(hw)));
  const size_t chunks = (n + grain - 1) / grain;
  if (hw <= 1 || chunks <= 1) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  const std::function<void(size_t)> fn = std::ref(f);
  pool.run(n, grain, fn);
}

using gdl::Adj;
using gdl::LigView;
using gdl::adjacency;
using gdl::reachable;
using gdl::validate;
using gdl::validation_message;
using gdl::view_of;

// ------------------------------------------------------------------ device arena
struct Arena {
  size_t off = 0;
  template <class T>
  size_t take(size_t count) {
    off = (off + 255) & ~size_t(255);
    const size_t at = off;
    off += count * sizeof(T);
    return at;
  }
};

int upload_params(gd_ctx* ctx) {
  // Rotation grid (geometry.cpp:16-34), FP64 with libm, plus FP32 rows of R/spacing.
  const gd_params& p = ctx->params;
  const uint32_t* st = p.rotation_steps;
  const uint64_t G = uint64_t(st[0]) * st[1] * st[2];
  std::vector<double4> grid(G);
  ctx->grid_host.assign(4 * G, 0.0);
  uint64_t at = 0;
  for (unsigned i = 0; i < st[0]; ++i) {
    const double alpha = gdh::kTwoPi * static_cast<double>(i) / static_cast<double>(st[0]);
    for (unsigned j = 0; j < st[1]; ++j) {
      const double beta = st[1] == 1 ? 0.0 : gdh::kPi * static_cast<double>(j) / static_cast<double>(st[1] - 1);
      for (unsigned k = 0; k < st[2]; ++k) {
        const double gamma = gdh::kTwoPi * static_cast<double>(k) / static_cast<double>(st[2]);
        const gdh::Q q = gdh::from_euler_zyz(alpha, beta, gamma);
        grid[at] = make_double4(q.w, q.x, q.y, q.z);
        ctx->grid_host[4 * at] = q.w;
        ctx->grid_host[4 * at + 1] = q.x;
        ctx->grid_host[4 * at + 2] = q.y;
        ctx->grid_host[4 * at + 3] = q.z;
        ++at;
      }
    }
  }
  // dihedral_step angles k * (2pi/S) and about_axis's (cos, sin) of the half angle
  // (docking.cpp:129,133; geometry.hpp:46-50; molecule.cpp:160).
  const uint32_t S = p.dihedral_steps;
  std::vector<double4> dtab(std::max<uint32_t>(S, 1));
  std::vector<float2> dtab_f(std::max<uint32_t>(S, 1));
  const double delta = gdh::kTwoPi / static_cast<double>(S);
  for (uint32_t k = 0; k < S; ++k) {
    const double angle = delta * static_cast<double>(k);
    const double half = 0.5 * angle;
    dtab[k] = make_double4(std::cos(half), std::sin(half), angle, 0.0);
    dtab_f[k] = make_float2(float(std::cos(half)), float(std::sin(half)));
  }
  cudaFree(ctx->d_grid);
  cudaFree(ctx->d_grid_f);
  cudaFree(ctx->d_dtab);
  cudaFree(ctx->d_dtab_f);
  ctx->d_grid = nullptr;
  ctx->d_grid_f = nullptr;
  ctx->d_dtab = nullptr;
  ctx->d_dtab_f = nullptr;
  GD_CUDA(ctx, cudaMalloc(&ctx->d_grid, sizeof(double4) * std::max<uint64_t>(G, 1)));
  GD_CUDA(ctx, cudaMalloc(&ctx->d_grid_f, sizeof(float4) * 3 * std::max<uint64_t>(G, 1)));
  GD_CUDA(ctx, cudaMalloc(&ctx->d_dtab, sizeof(double4) * dtab.size()));
  GD_CUDA(ctx, cudaMalloc(&ctx->d_dtab_f, sizeof(float2) * dtab_f.size()));
  GD_CUDA(ctx, cudaMemcpy(ctx->d_grid, grid.data(), sizeof(double4) * G, cudaMemcpyHostToDevice));
  GD_CUDA(ctx, cudaMemcpy(ctx->d_dtab, dtab.data(), sizeof(double4) * dtab.size(), cudaMemcpyHostToDevice));
  GD_CUDA(ctx, cudaMemcpy(ctx->d_dtab_f, dtab_f.data(), sizeof(float2) * dtab_f.size(), cudaMemcpyHostToDevice));
  ctx->G = uint32_t(G);
  return GD_OK;
}

// FP32 rotation rows R/spacing for the coarse path (depends on pocket spacing and grid).
int upload_grid_f(gd_ctx* ctx) {
  const uint32_t G = ctx->G;
  std::vector<float4> rows(3 * size_t(G));
  const double inv = 1.0 / ctx->spacing;
  for (uint32_t g = 0; g < G; ++g) {
    const double w = ctx->grid_host[4 * g], x = ctx->grid_host[4 * g + 1], y = ctx->grid_host[4 * g + 2],
                 z = ctx->grid_host[4 * g + 3];
    const double m[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                            {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                            {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    for (int r = 0; r < 3; ++r) {
      rows[3 * g + r] = make_float4(float(m[r][0] * inv), float(m[r][1] * inv), float(m[r][2] * inv), 0.f);
    }
  }
  GD_CUDA(ctx, cudaMemcpy(ctx->d_grid_f, rows.data(), sizeof(float4) * rows.size(), cudaMemcpyHostToDevice));
  // frames F_jk = Ry(beta_j) Rz(gamma_k) / spacing: R_g = Rz(alpha_i) F_jk for g = (i*b + j)*c + k
  const uint32_t* st = ctx->params.rotation_steps;
  const uint32_t nf = st[1] * st[2];
  std::vector<float4> fr(3 * size_t(std::max<uint32_t>(nf, 1)));
  for (unsigned j = 0; j < st[1]; ++j) {
    const double beta = st[1] == 1 ? 0.0 : gdh::kPi * static_cast<double>(j) / static_cast<double>(st[1] - 1);
    for (unsigned k = 0; k < st[2]; ++k) {
      const double gamma = gdh::kTwoPi * static_cast<double>(k) / static_cast<double>(st[2]);
      const gdh::Q q = gdh::compose(gdh::about_axis(0.0, 1.0, 0.0, beta), gdh::about_axis(0.0, 0.0, 1.0, gamma));
      const double w = q.w, x = q.x, y = q.y, z = q.z;
      const double m[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                              {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                              {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
      const size_t f = size_t(j) * st[2] + k;
      for (int r = 0; r < 3; ++r)
        fr[3 * f + r] = make_float4(float(m[r][0] * inv), float(m[r][1] * inv), float(m[r][2] * inv), 0.f);
    }
  }
  cudaFree(ctx->d_frames);
  ctx->d_frames = nullptr;
  GD_CUDA(ctx, cudaMalloc(&ctx->d_frames, sizeof(float4) * fr.size()));
  GD_CUDA(ctx, cudaMemcpy(ctx->d_frames, fr.data(), sizeof(float4) * fr.size(), cudaMemcpyHostToDevice));
  // Twin frames (the coarse alignment screens each distinct rotation once): frame f
  // is a twin of an earlier kept frame f0 with alpha shift s when F_f = Rz(alpha_s) F_f0, so that
  // R(i, f) = Rz(alpha_i) F_f = R((i + s) mod a, f0). On the default 16 x 16 x 8 grid the beta = 0 and
  // beta = pi rows collapse this way (14 of 128 frames; the 2048 rotations hold 1840 distinct
  // quaternions). Table layout (u32): [0, nf) per frame: (twin list offset << 8) | twin count for a
  // kept frame, 0xffffffff for a twin; [nf, nf + n_kept) the kept frames in index order; then the
  // twin lists, (f' | s << 16). The exact FP64 re-scoring in K1b scores every twin itself.
  {
    const uint32_t na = st[0];
    std::vector<std::array<double, 9>> fm(nf);
    for (unsigned j = 0; j < st[1]; ++j) {
      const double beta = st[1] == 1 ? 0.0 : gdh::kPi * static_cast<double>(j) / static_cast<double>(st[1] - 1);
      for (unsigned k = 0; k < st[2]; ++k) {
        const double gamma = gdh::kTwoPi * static_cast<double>(k) / static_cast<double>(st[2]);
        const gdh::Q q = gdh::compose(gdh::about_axis(0.0, 1.0, 0.0, beta), gdh::about_axis(0.0, 0.0, 1.0, gamma));
        const double w = q.w, x = q.x, y = q.y, z = q.z;
        fm[size_t(j) * st[2] + k] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                                     2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                                     2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
      }
    }
    std::vector<int32_t> rep(nf, -1), shift(nf, 0);
    std::vector<uint32_t> kept;
    for (uint32_t f = 0; f < nf; ++f) {
      for (uint32_t f0 : kept) {
        for (uint32_t sh = 0; sh < na && rep[f] < 0; ++sh) {
          const double al = gdh::kTwoPi * static_cast<double>(sh) / static_cast<double>(na);
          const double c = std::cos(al), sn = std::sin(al);
          const auto& m0 = fm[f0];
          double err = 0.0;
          for (int col = 0; col < 3; ++col) {  // Rz(alpha) F_f0 against F_f
            const double r0 = c * m0[col] - sn * m0[3 + col], r1 = sn * m0[col] + c * m0[3 + col], r2 = m0[6 + col];
            err = std::max({err, std::fabs(r0 - fm[f][col]), std::fabs(r1 - fm[f][3 + col]), std::fabs(r2 - fm[f][6 + col])});
          }
          if (err < 1e-12) {
            rep[f] = int32_t(f0);
            shift[f] = int32_t(sh);
          }
        }
        if (rep[f] >= 0) break;
      }
      if (rep[f] < 0) kept.push_back(f);
    }
    // K1a work units (kept frame, first of two quarter-turn groups c0), ordered by (gamma, c0, beta):
    // consecutive lanes take neighbouring beta rows, so the 8 lanes of one shared-memory phase
    // sample nearby points and share cells (fewer bank conflicts; tools/bank_sim.py: 9.4 -> 6.5
    // wavefronts per LDS.128 on C2).
    const uint32_t nq = na / 4;
    std::vector<uint32_t> units;
    for (uint32_t k = 0; k < st[2]; ++k)
      for (uint32_t c0 = 0; c0 < std::max<uint32_t>(nq, 1); c0 += gdk::k1a_qt_groups())
        for (uint32_t j = 0; j < st[1]; ++j) {
          const uint32_t f = j * st[2] + k;
          if (std::find(kept.begin(), kept.end(), f) != kept.end()) units.push_back(f | (c0 << 16));
        }
    std::vector<uint32_t> tab(nf + units.size(), 0u);
    for (uint32_t i = 0; i < units.size(); ++i) tab[nf + i] = units[i];
    for (uint32_t f0 : kept) {
      uint32_t cnt = 0;
      const uint32_t off = uint32_t(tab.size());
      for (uint32_t f = 0; f < nf; ++f)
        if (rep[f] == int32_t(f0)) {
          tab.push_back(f | (uint32_t(shift[f]) << 16));
          ++cnt;
        }
      tab[f0] = (off << 8) | cnt;
    }
    for (uint32_t f = 0; f < nf; ++f)
      if (rep[f] >= 0) tab[f] = 0xffffffffu;
    if (const char* env = std::getenv("GD_NO_TWINS"))  // experiments: screen every frame, frame-major units
      if (env[0] == '1') {
        units.clear();
        for (uint32_t f = 0; f < nf; ++f)
          for (uint32_t c0 = 0; c0 < std::max<uint32_t>(nq, 1); c0 += gdk::k1a_qt_groups()) units.push_back(f | (c0 << 16));
        tab.assign(nf + units.size(), 0u);
        for (uint32_t i = 0; i < units.size(); ++i) tab[nf + i] = units[i];
      }
    ctx->n_kept = uint32_t(units.size());  // K1a work units
    ctx->n_twin_frames = nf - uint32_t(kept.size());
    if (const char* env = std::getenv("GD_NO_TWINS"))
      if (env[0] == '1') ctx->n_twin_frames = 0;
    cudaFree(ctx->d_frame_tab);
    ctx->d_frame_tab = nullptr;
    GD_CUDA(ctx, cudaMalloc(&ctx->d_frame_tab, sizeof(uint32_t) * tab.size()));
    GD_CUDA(ctx, cudaMemcpy(ctx->d_frame_tab, tab.data(), sizeof(uint32_t) * tab.size(), cudaMemcpyHostToDevice));
  }
  return GD_OK;
}

// The pocket cells as an L2-persisting, read-only window on every stream of the context: they
// are re-read by every warp of every work item, so they should never be evicted by the batch
// traffic (C5's 47^3 grid does not fit shared memory and is read through L1/L2). Best effort: a
// device without persisting L2 simply keeps the normal policy.
void apply_l2_window(gd_ctx* ctx, void* base, size_t bytes) {
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
  if (max_persist <= 0 || max_window <= 0 || !base || bytes == 0) return;
  const size_t persist = std::min(bytes, size_t(max_persist));
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.base_ptr = base;
  v.accessPolicyWindow.num_bytes = std::min(bytes, size_t(max_window));
  v.accessPolicyWindow.hitRatio = 1.0f;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  for (cudaStream_t st : {ctx->stream, ctx->sa, ctx->sb})
    if (st && cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) cudaGetLastError();
  for (auto& sl : ctx->slot)
    if (sl.stream && cudaStreamSetAttribute(sl.stream, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess)
      cudaGetLastError();
}

DevPocket dev_pocket(const gd_ctx* ctx) {
  DevPocket pk{};
  pk.field = ctx->d_field;
  pk.cells = ctx->d_cells;
  for (int i = 0; i < 3; ++i) {
    pk.dims[i] = ctx->dims[i];
    pk.cell_dims[i] = ctx->dims[i] - 1;
    pk.origin[i] = ctx->origin[i];
    pk.maxc[i] = static_cast<double>(ctx->dims[i] - 1);
  }
  pk.spacing = ctx->spacing;
  pk.inv_spacing = 1.0 / ctx->spacing;
  pk.inv_spacing_f = float(1.0 / ctx->spacing);
  pk.q_eps = ctx->q_eps;
  pk.max_step = ctx->max_step;
  pk.coarse_scale = 1.0f;
  pk.dz_bias = ctx->dz_bias;
  pk.field_f = ctx->d_field_f;
  pk.f_dummy = ctx->dims[0] * ctx->dims[1] * ctx->dims[2];
  pk.f_count = ctx->f_count;
  pk.q_eps_f = ctx->q_eps_f;
  return pk;
}

DevParams dev_params(const gd_ctx* ctx) {
  DevParams pr{};
  pr.grid = ctx->d_grid;
  pr.grid_f = ctx->d_grid_f;
  pr.dtab = ctx->d_dtab;
  pr.dtab_f = ctx->d_dtab_f;
  pr.frames = ctx->d_frames;
  pr.frame_tab = ctx->d_frame_tab;
  pr.n_kept = ctx->n_kept;
  pr.n_twin_frames = ctx->n_twin_frames;
  for (int i = 0; i < 3; ++i) pr.steps[i] = ctx->params.rotation_steps[i];
  for (uint32_t i = 0; i < 16; ++i) {
    const double alpha = i < pr.steps[0] ? gdh::kTwoPi * static_cast<double>(i) / static_cast<double>(pr.steps[0]) : 0.0;
    pr.acs[i] = make_float2(float(std::cos(alpha)), float(std::sin(alpha)));
  }
  pr.n_restarts = ctx->params.n_restarts;
  pr.reps = ctx->params.num_repetitions;
  pr.G = ctx->G;
  pr.S = ctx->params.dihedral_steps;
  pr.clash = ctx->params.clash_factor;
  pr.clash_f = float(ctx->params.clash_factor);
  pr.mode = ctx->mode;
  return pr;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

gd_params gd_default_params(void) {
  gd_params p;
  p.n_restarts = 32;
  p.num_repetitions = 3;
  p.rotation_steps[0] = 16;
  p.rotation_steps[1] = 16;
  p.rotation_steps[2] = 8;
  p.dihedral_steps = 36;
  p.clash_factor = 0.75;
  p.seed = 0;
  return p;
}

const char* gd_version(void) { return "geodock_b200 0.1 (sm_100a)"; }

uint64_t gd_count_score_calls(const gd_params* p, uint64_t n_rotamers) {  // docking.cpp:44-50
  const uint64_t grid = uint64_t(p->rotation_steps[0]) * p->rotation_steps[1] * p->rotation_steps[2];
  return uint64_t(p->n_restarts) * (grid + uint64_t(p->num_repetitions) * n_rotamers * p->dihedral_steps);
}

int gd_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

int gd_create(int device, gd_ctx** out) {
  if (!out) return GD_ERR_ARGUMENT;
  *out = nullptr;
  auto* ctx = new gd_ctx();
  HostPool::live_contexts.fetch_add(1);
  ctx->device = device;
  ctx->params = gd_default_params();
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->n_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_stats, sizeof(unsigned long long) * 32);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_error, sizeof(int) * 2);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_counter, sizeof(unsigned int) * 4);
  for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&ctx->ev[i]);
  for (int i = 0; i < kSlots && e == cudaSuccess; ++i) {
    e = cudaStreamCreateWithFlags(&ctx->slot[i].stream, cudaStreamNonBlocking);
    for (cudaEvent_t* ev : {&ctx->slot[i].in, &ctx->slot[i].done})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    for (cudaEvent_t* ev : {&ctx->slot[i].a0, &ctx->slot[i].mid, &ctx->slot[i].k})
      if (e == cudaSuccess) e = cudaEventCreate(ev);
  }
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->run0);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->run1);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->sa, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->sb, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    gd_destroy(ctx);  // releases whatever was created before the failure (streams, events, buffers)
    return GD_ERR_CUDA;
  }
  ctx->have_params = upload_params(ctx) == GD_OK;
  *out = ctx;
  return ctx->have_params ? GD_OK : GD_ERR_CUDA;
}

void gd_destroy(gd_ctx* ctx) {
  if (!ctx) return;
  HostPool::live_contexts.fetch_sub(1);
  cudaSetDevice(ctx->device);
  cudaFree(ctx->d_field);
  cudaFree(ctx->d_cells);
  cudaFree(ctx->d_field_f);
  cudaFree(ctx->d_grid);
  cudaFree(ctx->d_grid_f);
  cudaFree(ctx->d_frames);
  cudaFree(ctx->d_frame_tab);
  cudaFree(ctx->d_dtab);
  cudaFree(ctx->d_dtab_f);
  cudaFree(ctx->d_stats);
  cudaFree(ctx->d_error);
  cudaFree(ctx->d_counter);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& sl : ctx->slot) {
    if (sl.h_in) cudaFreeHost(sl.h_in);
    if (sl.h_out) cudaFreeHost(sl.h_out);
    cudaFree(sl.d_arena);
    for (cudaEvent_t ev : {sl.in, sl.mid, sl.k, sl.done, sl.a0})
      if (ev) cudaEventDestroy(ev);
    if (sl.stream) cudaStreamDestroy(sl.stream);
  }
  if (ctx->run0) cudaEventDestroy(ctx->run0);
  if (ctx->run1) cudaEventDestroy(ctx->run1);
  if (ctx->sa) cudaStreamDestroy(ctx->sa);
  if (ctx->sb) cudaStreamDestroy(ctx->sb);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx->pool;
  delete ctx;
}

const char* gd_last_error(const gd_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* gd_stream(gd_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int gd_set_mode(gd_ctx* ctx, int mode) {
  if (!ctx) return GD_ERR_ARGUMENT;
  if ((mode & 0xff) != GD_MODE_FAST && (mode & 0xff) != GD_MODE_EXACT) {
    return set_err(ctx, GD_ERR_ARGUMENT, "unknown mode");
  }
  ctx->mode = mode;
  return GD_OK;
}

int gd_set_params(gd_ctx* ctx, const gd_params* p) {
  if (!ctx || !p) return GD_ERR_ARGUMENT;
  if (!p->rotation_steps[0] || !p->rotation_steps[1] || !p->rotation_steps[2]) {
    return set_err(ctx, GD_ERR_CONTRACT, "rotation grid steps must all be >= 1");  // geometry.cpp:18-20
  }
  cudaSetDevice(ctx->device);
  ctx->params = *p;
  ctx->have_params = false;
  int rc = upload_params(ctx);
  if (rc != GD_OK) return rc;
  if (ctx->have_pocket) rc = upload_grid_f(ctx);
  ctx->have_params = rc == GD_OK;
  return rc;
}

int gd_set_pocket(gd_ctx* ctx, const uint32_t dims[3], const double origin[3], double spacing,
                  const double* field) {
  if (!ctx || !dims || !origin || !field) return GD_ERR_ARGUMENT;
  if (dims[0] < 2 || dims[1] < 2 || dims[2] < 2) return set_err(ctx, GD_ERR_CONTRACT, "pocket dims must be >= 2");
  if (!(spacing > 0.0)) return set_err(ctx, GD_ERR_CONTRACT, "pocket spacing must be > 0");
  cudaSetDevice(ctx->device);
  const size_t nv = size_t(dims[0]) * dims[1] * dims[2];
  cudaFree(ctx->d_field);
  cudaFree(ctx->d_cells);
  ctx->d_field = nullptr;
  ctx->d_cells = nullptr;
  GD_CUDA(ctx, cudaMalloc(&ctx->d_field, nv * sizeof(double)));
  GD_CUDA(ctx, cudaMemcpy(ctx->d_field, field, nv * sizeof(double), cudaMemcpyHostToDevice));

  // Coarse-path cells: for every grid cell (ix,iy,iz) < dims-1 and each of its two
  // y-edges j, the bilinear form in (fx, fz) of the face's corners v(x+a, y+j, z+b):
  //   v = C0 + fz dC + fx (D0 + fz dD),
  // quantised with error feedback (each field absorbs the rounding of the ones before it, so every
  // corner is within half a step of its own field), two words per edge:
  //   word 2j   = (0x8000 | round(32768 C0)) | round(16384 (1 - dC)) << 16
  //   word 2j+1 = round(16384 (1 + D0))      | dD field << 16
  // with the dD field round(16384 (1 - dD)) (B = 3) or 0x8000 | round(8192 (2 - dD)) (B = 6, when a
  // second difference leaves (-1, 1]). The kernel's byte permutes decode 1 + C0, dC - 3, 3 + D0 and
  // dD - B (cell_lerp_b). One extra dummy cell (all fields zero) at index cx*cy*cz evaluates to ~0
  // for any fractions: samples outside the grid read it.
  const uint32_t cx = dims[0] - 1, cy = dims[1] - 1, cz = dims[2] - 1;
  std::vector<uint4> cells(size_t(cx) * cy * cz + 1);
  double max_step = 0.0;  // largest |v(i+1) - v(i)| along any axis: Lipschitz bound per cell
  double q_err = 0.0;     // largest |decoded - v| over all face corners: quantisation bound
  auto at = [&](uint32_t x, uint32_t y, uint32_t z) { return field[(size_t(z) * dims[1] + y) * dims[0] + x]; };
  auto clamp01 = [](double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); };
  auto q15 = [](double v) { return std::min(32767L, std::max(0L, std::lround(v))); };
  struct Face {
    long uc, udc, ud0;
    double c0, dc, d0, rest;  // quantised C0, dC, D0; the second difference dD still to quantise
    double v[4];              // corners (fx, fz) = (0,0), (1,0), (0,1), (1,1)
  };
  auto face = [&](uint32_t x, uint32_t y, uint32_t z) -> Face {
    Face f{};
    f.v[0] = clamp01(at(x, y, z));
    f.v[1] = clamp01(at(x + 1, y, z));
    f.v[2] = clamp01(at(x, y, z + 1));
    f.v[3] = clamp01(at(x + 1, y, z + 1));
    f.uc = q15(f.v[0] * 32768.0);
    f.c0 = double(f.uc) / 32768.0;
    f.ud0 = q15((1.0 + (f.v[1] - f.c0)) * 16384.0);
    f.d0 = double(f.ud0) / 16384.0 - 1.0;
    f.udc = q15((1.0 - (f.v[2] - f.c0)) * 16384.0);
    f.dc = 1.0 - double(f.udc) / 16384.0;
    f.rest = f.v[3] - f.c0 - f.d0 - f.dc;
    return f;
  };
  // pass 1: the dD range decides B
  bool wide = false;
  for (uint32_t z = 0; z < cz && !wide; ++z)
    for (uint32_t y = 0; y < dims[1] && !wide; ++y)
      for (uint32_t x = 0; x < cx; ++x) {
        const double r = face(x, y, z).rest;
        if (!(r > -0.99 && r <= 0.99)) {
          wide = true;
          break;
        }
      }
  auto words = [&](uint32_t x, uint32_t y, uint32_t z, uint32_t& w0, uint32_t& w1) {
    const Face f = face(x, y, z);
    long udd;
    double dd;
    if (!wide) {
      udd = q15((1.0 - f.rest) * 16384.0);
      dd = 1.0 - double(udd) / 16384.0;
    } else {
      udd = q15((2.0 - f.rest) * 8192.0);
      dd = 2.0 - double(udd) / 8192.0;
      udd |= 0x8000L;
    }
    const double got[4] = {f.c0, f.c0 + f.d0, f.c0 + f.dc, f.c0 + f.d0 + f.dc + dd};
    for (int c = 0; c < 4; ++c) q_err = std::max(q_err, std::fabs(got[c] - f.v[c]));
    w0 = (0x8000u | uint32_t(f.uc)) | (uint32_t(f.udc) << 16);
    w1 = uint32_t(f.ud0) | (uint32_t(udd) << 16);
  };
  for (uint32_t z = 0; z < cz; ++z)
    for (uint32_t y = 0; y < cy; ++y)
      for (uint32_t x = 0; x < cx; ++x) {
        uint4 w;
        words(x, y, z, w.x, w.y);
        words(x, y + 1, z, w.z, w.w);
        cells[(size_t(z) * cy + y) * cx + x] = w;
        for (int c = 0; c < 8; ++c) {
          const double v0 = at(x + (c & 1), y + ((c >> 1) & 1), z + ((c >> 2) & 1));
          if (!(c & 1)) max_step = std::max(max_step, std::fabs(at(x + 1, y + ((c >> 1) & 1), z + ((c >> 2) & 1)) - v0));
          if (!(c & 2)) max_step = std::max(max_step, std::fabs(at(x + (c & 1), y + 1, z + ((c >> 2) & 1)) - v0));
          if (!(c & 4)) max_step = std::max(max_step, std::fabs(at(x + (c & 1), y + ((c >> 1) & 1), z + 1) - v0));
        }
      }
  {  // dummy: C0 = dC = D0 = dD = 0
    const uint32_t w0 = 0x8000u | (16384u << 16);
    const uint32_t w1 = 16384u | ((wide ? (0x8000u | 16384u) : 16384u) << 16);
    cells.back() = make_uint4(w0, w1, w0, w1);
  }
  ctx->dz_bias = wide ? 6.0f : 3.0f;
  bool in_range = true;
  for (size_t i = 0; i < nv; ++i) in_range &= (field[i] >= 0.0 && field[i] <= 1.0);
  {  // K1b's FP32 field: the clamped values, then zeros for the 8 corners of a sample outside
    const size_t tail = size_t(dims[0]) * dims[1] + dims[0] + 2;
    std::vector<float> ff((nv + tail + 3) & ~size_t(3), 0.f);
    double qf = 0.0;
    for (size_t i = 0; i < nv; ++i) {
      const double v = clamp01(field[i]);
      ff[i] = float(v);
      qf = std::max(qf, std::fabs(double(ff[i]) - v));
    }
    cudaFree(ctx->d_field_f);
    ctx->d_field_f = nullptr;
    GD_CUDA(ctx, cudaMalloc(&ctx->d_field_f, ff.size() * sizeof(float)));
    GD_CUDA(ctx, cudaMemcpy(ctx->d_field_f, ff.data(), ff.size() * sizeof(float), cudaMemcpyHostToDevice));
    ctx->f_count = uint32_t(ff.size());
    ctx->q_eps_f = float(qf * (1.0 + 1e-6) + 1e-12);
  }
  GD_CUDA(ctx, cudaMalloc(&ctx->d_cells, cells.size() * sizeof(uint4)));
  GD_CUDA(ctx, cudaMemcpy(ctx->d_cells, cells.data(), cells.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  // Coarse error model: quantisation q_err per sample (each face's decoded form
  // is the bilinear interpolant of its decoded corners, the y-lerp a convex combination); the
  // kernel adds 3 * max_step * (its FP32 position bound). A field outside [0,1] breaks the quantiser, so the fast path is disabled for it (q_eps = inf ->
  // exact kernel).
  ctx->q_eps = in_range ? float(q_err * (1.0 + 1e-6)) : INFINITY;
  apply_l2_window(ctx, ctx->d_cells, cells.size() * sizeof(uint4));
  ctx->max_step = float(max_step);
  for (int i = 0; i < 3; ++i) {
    ctx->dims[i] = dims[i];
    ctx->origin[i] = origin[i];
  }
  ctx->spacing = spacing;
  ctx->have_pocket = true;
  return upload_grid_f(ctx);
}

int gd_validate_ligand(const gd_library* lib, uint32_t l, char* msg, uint32_t cap) {
  if (!lib || l >= lib->n_ligands) return -1;
  const std::vector<std::string> v = validate(view_of(lib, l));
  std::string all;
  for (const auto& s : v) all += s + "\n";
  if (msg && cap) std::snprintf(msg, cap, "%s", all.c_str());
  return int(v.size());
}

int gd_moving_set(const gd_library* lib, uint32_t l, uint32_t r, uint32_t* out, uint32_t* out_len) {
  if (!lib || l >= lib->n_ligands || !out || !out_len) return GD_ERR_ARGUMENT;
  const LigView v = view_of(lib, l);
  if (!validate(v).empty()) return GD_ERR_INVALID_LIGAND;
  if (r >= v.nr) return GD_ERR_CONTRACT;
  const Adj adj = adjacency(v);
  std::vector<char> seen;
  std::vector<uint32_t> stack;
  reachable(adj, v.n, v.rots[2 * r + 1], v.rots[2 * r], v.rots[2 * r + 1], seen, stack);
  uint32_t k = 0;
  for (uint32_t a = 0; a < v.n; ++a)
    if (seen[a]) out[k++] = a;
  *out_len = k;
  return GD_OK;
}

}  // extern "C"

namespace {

// ------------------------------------------------------------------ batch layout / packing
// One packed batch lives in one device arena: [0, host_bytes) is packed on the host and uploaded,
// the rest is per-restart scratch and per-ligand results.

Layout plan_layout(const gd_library* lib, const gd_params& P) {
  Layout y;
  const uint32_t L = lib->n_ligands, N = P.n_restarts, reps = P.num_repetitions;
  y.L = L;
  y.A = L ? lib->atom_off[L] - lib->atom_off[0] : 0;
  y.Rt = L ? lib->rot_off[L] - lib->rot_off[0] : 0;
  y.mask_base.assign(L + 1, 0);
  y.adj_base.assign(L + 1, 0);
  for (uint32_t l = 0; l < L; ++l) {
    const uint32_t n = lib->atom_off[l + 1] - lib->atom_off[l];
    const uint32_t W = (n + 31) / 32;
    y.max_n = std::max(y.max_n, n);
    if (n <= gdk::kFastMaxAtoms) y.fast_max_n = std::max(y.fast_max_n, n);
    if (n <= gdk::kFastMaxAtoms) {
      const int c = n <= 32 ? 0 : (n <= 64 ? 1 : 2);
      y.class_max_n[c] = std::max(y.class_max_n[c], n);
    }
    y.mask_base[l + 1] = y.mask_base[l] + (lib->rot_off[l + 1] - lib->rot_off[l]) * W;
    y.adj_base[l + 1] = y.adj_base[l] + n * W;
  }
  y.n_items = size_t(L) * N;
  Arena ar;
  y.o_meta = ar.take<LigMeta>(L);
  y.o_atoms = ar.take<double4>(y.A);
  y.o_start = ar.take<double4>(2 * y.n_items);
  y.o_rots = ar.take<uint2>(y.Rt);
  y.o_dih0 = ar.take<double>(y.Rt);
  y.o_masks = ar.take<uint32_t>(y.mask_base[L]);
  y.o_adj = ar.take<uint32_t>(y.adj_base[L]);
  y.o_dfs = ar.take<uint16_t>(y.A);
  y.o_rdfs = ar.take<ushort4>(y.Rt);
  y.o_adjd = ar.take<uint32_t>(y.adj_base[L]);
  y.host_bytes = ar.off;
  y.o_cand = ar.take<uint16_t>(y.n_items * gdk::kAlignCand);
  y.o_ncand = ar.take<int32_t>(y.n_items);
  y.o_rs_score = ar.take<double>(y.n_items);
  y.o_rs_ascore = ar.take<double>(y.n_items);
  y.o_rs_aidx = ar.take<uint32_t>(y.n_items);
  y.o_rs_stepk = ar.take<int32_t>(size_t(y.Rt) * N * reps);
  y.o_rs_pose = ar.take<double>(size_t(y.A) * N * 3);  // K1r -> K1b: aligned FP64 pose per restart
  y.o_rs_es = ar.take<double>(size_t(y.A) * N);        // and its exact per-atom samples
  y.o_rs_ext = ar.take<float>(y.n_items);
  y.o_slow = ar.take<uint32_t>(y.n_items);  // K1b -> FP64 kernel: restarts handed over
  y.o_best = ar.take<double>(L);
  y.o_brs = ar.take<uint32_t>(L);
  y.o_fxyz = ar.take<double>(size_t(y.A) * 3);
  y.o_fdih = ar.take<double>(y.Rt);
  y.o_ctr = ar.take<unsigned int>(20);  // work counters: [0..3] exact / one-class, [4 c ..] class c, [16..] K1a NS = 8
  y.o_order = ar.take<uint32_t>(y.n_items);
  y.o_ord_scr = ar.take<uint32_t>(3 * y.n_items);
  y.ord_tmp_bytes = gdk::order_tmp_bytes(uint32_t(y.n_items));
  y.o_ord_tmp = ar.take<unsigned char>(y.ord_tmp_bytes);
  y.total = ar.off + 256;
  return y;
}

// Validation of ligands [l0, l1) in library order (dock_ligand throws before any work,
// docking.cpp:239-240; run_screening reports the first failing task, pipeline.cpp:233).
int validate_range(gd_ctx* ctx, const gd_library* lib, uint32_t l0, uint32_t l1) {
  std::vector<uint8_t> bad(l1 - l0, 0);
  parallel_for(ctx, l1 - l0, 0, [&](size_t i) {
    const LigView v = view_of(lib, uint32_t(l0 + i));
    bad[i] = (!validate(v).empty() || v.n > GD_MAX_ATOMS) ? 1u : 0u;
  });
  for (uint32_t l = l0; l < l1; ++l) {
    if (!bad[l - l0]) continue;
    const LigView v = view_of(lib, l);
    const auto viol = validate(v);
    if (!viol.empty()) return set_err(ctx, GD_ERR_INVALID_LIGAND, validation_message(v.name, viol));
    return set_err(ctx, GD_ERR_UNSUPPORTED, "ligand '" + std::string(v.name) + "' has " + std::to_string(v.n) +
                                                " atoms; this build supports up to " + std::to_string(GD_MAX_ATOMS));
  }
  return GD_OK;
}

// bump_check's clash-factor contract (scoring.cpp:48-50) fires at the first bump_check, i.e. in the
// first dihedral step of the first ligand that has rotamers (and only when restarts, repetitions
// and dihedral steps are all non-zero). dock_ligand validates that ligand before (docking.cpp:239-240)
// and run_screening validates every task before docking it (pipeline.cpp:233): an invalid ligand
// up to and including that one is reported first.
int check_contract(gd_ctx* ctx, const gd_library* lib) {
  const gd_params& P = ctx->params;
  if (!(P.n_restarts && P.num_repetitions && P.dihedral_steps)) return GD_OK;
  if (P.clash_factor > 0.0 && P.clash_factor <= 1.0) return GD_OK;
  const uint32_t L = lib->n_ligands;
  for (uint32_t l = 0; l < L; ++l) {
    if (lib->rot_off[l + 1] == lib->rot_off[l]) continue;
    const int rc = validate_range(ctx, lib, 0, l + 1);
    if (rc != GD_OK) return rc;
    return set_err(ctx, GD_ERR_CONTRACT, "clash_factor must lie in (0, 1]");
  }
  return GD_OK;
}

// Per-thread scratch of the packer (no heap traffic per ligand once warm).
struct PackScratch {
  std::vector<uint32_t> start, nbr, fill, order, tin, low, par, sz, cover, msize;
  std::vector<std::pair<uint32_t, uint32_t>> st;
};

// Iterative DFS from `root` over the CSR graph, neighbours in CSR order: preorder (order, tin),
// parent, subtree size and low-link (lowest preorder index reachable from the subtree by one
// non-parent edge; every edge to the parent is skipped, so parallel bonds count as one edge, as
// in reachable(), molecule.cpp:22-41, which drops all (i, j) edges). Returns the atoms visited.
inline uint32_t dfs_tree(PackScratch& g, uint32_t n, uint32_t root) {
  constexpr uint32_t NONE = ~0u;
  g.tin.assign(n, NONE);
  g.low.resize(n);
  g.par.resize(n);
  g.sz.resize(n);
  g.order.clear();
  g.st.clear();
  g.tin[root] = g.low[root] = 0;
  g.par[root] = NONE;
  g.order.push_back(root);
  g.st.push_back({root, g.start[root]});
  while (!g.st.empty()) {
    auto& top = g.st.back();
    const uint32_t u = top.first;
    if (top.second == g.start[u + 1]) {
      g.st.pop_back();
      g.sz[u] = uint32_t(g.order.size()) - g.tin[u];
      if (g.par[u] != NONE) g.low[g.par[u]] = std::min(g.low[g.par[u]], g.low[u]);
      continue;
    }
    const uint32_t w = g.nbr[top.second++];
    if (w == g.par[u]) continue;
    if (g.tin[w] == NONE) {
      g.par[w] = u;
      g.tin[w] = g.low[w] = uint32_t(g.order.size());
      g.order.push_back(w);
      g.st.push_back({w, g.start[w]});
    } else {
      g.low[u] = std::min(g.low[u], g.tin[w]);
    }
  }
  return uint32_t(g.order.size());
}

// Host SoA packing of a (rebased, atom_off[0] == 0) library into H[0, host_bytes), fused with
// validate_ligand (molecule.cpp:176-238): one pass over each ligand's graph builds its adjacency,
// checks it and derives the moving sets from the same DFS (the component of atom_j with the bond
// (i, j) removed is both the ring check and the moving set, molecule.cpp:88-98). Returns the index
// of the first ligand that fails validation (or exceeds GD_MAX_ATOMS) in library order, or -1;
// invalid ligands are not packed.
int64_t pack_library(const gd_ctx* ctx, const gd_library* lib, const Layout& y, unsigned char* H) {
  const gd_params& P = ctx->params;
  const uint32_t L = y.L, N = P.n_restarts;
  auto* meta = reinterpret_cast<LigMeta*>(H + y.o_meta);
  auto* atoms = reinterpret_cast<double4*>(H + y.o_atoms);
  auto* start = reinterpret_cast<double4*>(H + y.o_start);
  auto* rots = reinterpret_cast<uint2*>(H + y.o_rots);
  auto* dih0 = reinterpret_cast<double*>(H + y.o_dih0);
  auto* masks = reinterpret_cast<uint32_t*>(H + y.o_masks);
  auto* adjm = reinterpret_cast<uint32_t*>(H + y.o_adj);
  auto* dfs = reinterpret_cast<uint16_t*>(H + y.o_dfs);
  auto* rdfs = reinterpret_cast<ushort4*>(H + y.o_rdfs);
  auto* adjd = reinterpret_cast<uint32_t*>(H + y.o_adjd);
  const double lo[3] = {ctx->origin[0], ctx->origin[1], ctx->origin[2]};
  // Pocket::bounds_hi (scoring.hpp:32-36)
  const double hi[3] = {ctx->origin[0] + ctx->spacing * static_cast<double>(ctx->dims[0] - 1),
                        ctx->origin[1] + ctx->spacing * static_cast<double>(ctx->dims[1] - 1),
                        ctx->origin[2] + ctx->spacing * static_cast<double>(ctx->dims[2] - 1)};
  const uint32_t a0 = L ? lib->atom_off[0] : 0, r0 = L ? lib->rot_off[0] : 0;
  std::atomic<int64_t> first_bad{int64_t(L)};
  parallel_for(const_cast<gd_ctx*>(ctx), L, 0, [&](size_t li) {
    thread_local PackScratch tls;
    PackScratch& g = tls;  // one TLS lookup per ligand (-fPIC: every thread_local access is a call)
    const uint32_t l = uint32_t(li);
    const LigView v = view_of(lib, l);
    const uint32_t n = v.n, W = (n + 31) / 32;
    auto bad = [&] {
      int64_t cur = first_bad.load();
      while (int64_t(l) < cur && !first_bad.compare_exchange_weak(cur, int64_t(l))) {
      }
    };
    // ---- validate_ligand's checks (the message is rebuilt by validate() for the reported ligand)
    if (n == 0 || n > GD_MAX_ATOMS || v.nr > GD_MAX_ROTAMERS) return bad();
    for (uint32_t a = 0; a < n; ++a) {
      if (!(v.radius[a] > 0.0) || !std::isfinite(v.xyz[3 * a]) || !std::isfinite(v.xyz[3 * a + 1]) ||
          !std::isfinite(v.xyz[3 * a + 2]))
        return bad();
    }
    for (uint32_t e = 0; e < v.nb; ++e) {
      const uint32_t x = v.bonds[2 * e], z = v.bonds[2 * e + 1];
      if (x >= n || z >= n || x == z) return bad();
    }
    // adjacency lists (adjacency_lists, molecule.cpp:12-20), CSR in scratch
    g.start.assign(n + 1, 0);
    for (uint32_t e = 0; e < v.nb; ++e) {
      g.start[v.bonds[2 * e] + 1]++;
      g.start[v.bonds[2 * e + 1] + 1]++;
    }
    for (uint32_t i = 0; i < n; ++i) g.start[i + 1] += g.start[i];
    g.nbr.resize(g.start[n]);
    g.fill.assign(g.start.begin(), g.start.end() - 1);
    for (uint32_t e = 0; e < v.nb; ++e) {
      const uint32_t x = v.bonds[2 * e], z = v.bonds[2 * e + 1];
      g.nbr[g.fill[x]++] = z;
      g.nbr[g.fill[z]++] = x;
    }
    // One DFS from atom 0 (preorder, subtree sizes, low-links) answers every graph question of
    // validate_ligand / finalize_ligand: connectivity (molecule.cpp:214-222), and per rotamer the
    // ring check and the moving set (molecule.cpp:88-98). The component of atom_j with the (i, j)
    // bonds removed excludes atom_i iff (i, j) is a bridge, i.e. a tree edge (p, c) with
    // low[c] > tin[p]; it is then subtree(j) when j is the child, else everything but subtree(i),
    // a range (or the complement of one) of preorder positions.
    if (dfs_tree(g, n, 0) != n) return bad();  // bond graph is not connected
    LigMeta m{};
    m.atom_base = lib->atom_off[l] - a0;
    m.rot_base = lib->rot_off[l] - r0;
    m.mask_base = y.mask_base[l];
    m.adj_base = y.adj_base[l];
    m.n = uint16_t(n);
    m.nr = uint16_t(v.nr);
    g.cover.assign(n + 1, 0);  // difference array over preorder positions: in some moving set
    g.msize.resize(v.nr);
    for (uint32_t r = 0; r < v.nr; ++r) {
      const uint32_t i = v.rots[2 * r], j = v.rots[2 * r + 1];
      if (i >= n || j >= n) return bad();
      bool bonded = false;
      for (uint32_t e = g.start[i]; e < g.start[i + 1]; ++e) bonded |= g.nbr[e] == j;
      if (!bonded) return bad();
      const bool j_child = g.par[j] == i;
      const uint32_t c = j_child ? j : i, p = j_child ? i : j;
      if (!(g.par[c] == p && g.low[c] > g.tin[p])) return bad();  // does not disconnect the graph
      rots[m.rot_base + r] = make_uint2(i, j);
      dih0[m.rot_base + r] = lib->dihedrals ? lib->dihedrals[lib->rot_off[l] + r] : 0.0;
      uint32_t* mk = masks + m.mask_base + r * W;
      std::fill(mk, mk + W, 0u);
      const uint32_t s0 = g.tin[c], e0 = s0 + g.sz[c];
      auto mark = [&](uint32_t q0, uint32_t q1) {
        for (uint32_t q = q0; q < q1; ++q) mk[g.order[q] >> 5] |= 1u << (g.order[q] & 31);
        g.cover[q0]++;
        g.cover[q1]--;
      };
      if (j_child) {
        mark(s0, e0);
      } else {
        mark(0, s0);
        mark(e0, n);
      }
      g.msize[r] = j_child ? g.sz[c] : n - g.sz[c];
    }
    meta[l] = m;
    for (uint32_t a = 0; a < n; ++a) {
      atoms[m.atom_base + a] = make_double4(v.xyz[3 * a], v.xyz[3 * a + 1], v.xyz[3 * a + 2], v.radius[a]);
    }
    // bonded rows (Ligand::adjacency, molecule.cpp:80-86)
    uint32_t* adj_l = adjm + m.adj_base;
    std::fill(adj_l, adj_l + size_t(n) * W, 0u);
    for (uint32_t e = 0; e < v.nb; ++e) {
      const uint32_t x = v.bonds[2 * e], z = v.bonds[2 * e + 1];
      adj_l[x * W + (z >> 5)] |= 1u << (z & 31);
      adj_l[z * W + (x >> 5)] |= 1u << (x & 31);
    }
    // DFS preorder from an atom outside every moving set: each moving set (the component of atom_j
    // behind the bridge (i,j)) is then entered only through j and is exactly j's subtree, one
    // contiguous range [pos(j), pos(j) + |M|) — the layout the fast sweep's range loops need
    // (DESIGN.md §3.3). When atom 0 is outside every moving set (the usual case) the validation
    // DFS above is that preorder already; else it is rerun from the first such atom.
    {
      uint32_t root = n, run = 0;
      for (uint32_t q = 0; q < n && root == n; ++q) {
        run += g.cover[q];
        if (run == 0) root = g.order[q];
      }
      const bool ok = root < n && n <= 128;
      if (root < n && root != 0) dfs_tree(g, n, root);
      uint16_t* dl = dfs + m.atom_base;
      for (uint32_t q = 0; q < n; ++q) dl[g.order[q]] = uint16_t(q);
      for (uint32_t r = 0; r < v.nr; ++r) {
        const uint32_t i = v.rots[2 * r], j = v.rots[2 * r + 1];
        const uint32_t s0 = dl[j];
        rdfs[m.rot_base + r] = make_ushort4(uint16_t(s0), uint16_t(s0 + g.msize[r]), dl[i], 0);
      }
      uint32_t* ad = adjd + m.adj_base;
      std::fill(ad, ad + size_t(n) * W, 0u);
      for (uint32_t e = 0; e < v.nb; ++e) {
        const uint32_t x = dl[v.bonds[2 * e]], z = dl[v.bonds[2 * e + 1]];
        ad[x * W + (z >> 5)] |= 1u << (z & 31);
        ad[z * W + (x >> 5)] |= 1u << (x & 31);
      }
      meta[l].fast_ok = ok ? 1u : 0u;
      meta[l].npad = (n + 3) & ~3u;
    }
    // starting transforms (generate_starting_pose, docking.cpp:52-69): q and target per restart.
    const uint64_t lig_seed = gdh::mix_seed(P.seed, gdh::fnv1a64(v.name));
    for (uint32_t pid = 0; pid < N; ++pid) {
      gdh::SplitMix64 rng(gdh::mix_seed(lig_seed, pid));
      const gdh::Q q = gdh::random_rotation(rng);
      const double tx = rng.uniform(lo[0], hi[0]);
      const double ty = rng.uniform(lo[1], hi[1]);
      const double tz = rng.uniform(lo[2], hi[2]);
      const size_t it = size_t(l) * N + pid;
      start[2 * it] = make_double4(q.w, q.x, q.y, q.z);
      start[2 * it + 1] = make_double4(tx, ty, tz, 0.0);
    }
  });
  const int64_t fb = first_bad.load();
  return fb < int64_t(L) ? fb : -1;
}

// The reference's error for ligand l (known to be invalid or too large): ValidationError with
// validate_ligand's messages, else GD_ERR_UNSUPPORTED.
int report_invalid(gd_ctx* ctx, const gd_library* lib, uint32_t l) {
  const LigView v = view_of(lib, l);
  const auto viol = validate(v);
  if (!viol.empty()) return set_err(ctx, GD_ERR_INVALID_LIGAND, validation_message(v.name, viol));
  return set_err(ctx, GD_ERR_UNSUPPORTED, "ligand '" + std::string(v.name) + "' has " + std::to_string(v.n) +
                                              " atoms; this build supports up to " + std::to_string(GD_MAX_ATOMS));
}

// Device view of a packed batch in arena D (ctx-level stats / error flag, per-batch counters).
DevBatch bind_batch(const gd_ctx* ctx, const Layout& y, unsigned char* D, uint32_t lig_base = 0) {
  DevBatch d{};
  d.n_lig = y.L;
  d.lig_base = lig_base;
  d.n_atoms = y.A;
  d.n_rots = y.Rt;
  d.max_n = y.max_n;
  d.fast_max_n = y.fast_max_n;
  d.fast_min_n = 0;
  for (int c = 0; c < 3; ++c) d.class_max_n[c] = y.class_max_n[c];
  d.meta = reinterpret_cast<const LigMeta*>(D + y.o_meta);
  d.atoms = reinterpret_cast<const double4*>(D + y.o_atoms);
  d.start = reinterpret_cast<const double4*>(D + y.o_start);
  d.rots = reinterpret_cast<const uint2*>(D + y.o_rots);
  d.dih0 = reinterpret_cast<const double*>(D + y.o_dih0);
  d.masks = reinterpret_cast<const uint32_t*>(D + y.o_masks);
  d.adj = reinterpret_cast<const uint32_t*>(D + y.o_adj);
  d.dfs_pos = reinterpret_cast<const uint16_t*>(D + y.o_dfs);
  d.rdfs = reinterpret_cast<const ushort4*>(D + y.o_rdfs);
  d.adjd = reinterpret_cast<const uint32_t*>(D + y.o_adjd);
  d.rs_cand = reinterpret_cast<uint16_t*>(D + y.o_cand);
  d.rs_ncand = reinterpret_cast<int32_t*>(D + y.o_ncand);
  d.rs_score = reinterpret_cast<double*>(D + y.o_rs_score);
  d.rs_align_score = reinterpret_cast<double*>(D + y.o_rs_ascore);
  d.rs_align_index = reinterpret_cast<uint32_t*>(D + y.o_rs_aidx);
  d.rs_step_k = reinterpret_cast<int32_t*>(D + y.o_rs_stepk);
  d.rs_pose = reinterpret_cast<double*>(D + y.o_rs_pose);
  d.rs_es = reinterpret_cast<double*>(D + y.o_rs_es);
  d.rs_ext = reinterpret_cast<float*>(D + y.o_rs_ext);
  d.slow_items = reinterpret_cast<uint32_t*>(D + y.o_slow);
  d.best_score = reinterpret_cast<double*>(D + y.o_best);
  d.best_restart = reinterpret_cast<uint32_t*>(D + y.o_brs);
  d.final_xyz = reinterpret_cast<double*>(D + y.o_fxyz);
  d.final_dih = reinterpret_cast<double*>(D + y.o_fdih);
  d.work_counter = reinterpret_cast<unsigned int*>(D + y.o_ctr);
  d.slow_count = d.work_counter + 19;
  const bool ordered = y.n_items > 0 && !std::getenv("GD_NATURAL_ORDER");  // (A/B experiments)
  d.order = ordered ? reinterpret_cast<uint32_t*>(D + y.o_order) : nullptr;
  d.order_scratch = reinterpret_cast<uint32_t*>(D + y.o_ord_scr);
  d.order_tmp = D + y.o_ord_tmp;
  d.order_tmp_bytes = y.ord_tmp_bytes;
  d.error = ctx->d_error;
  d.stats = ctx->d_stats;
  return d;
}

int reset_device_status(gd_ctx* ctx, cudaStream_t s) {
  GD_CUDA(ctx, cudaMemsetAsync(ctx->d_error, 0, 2 * sizeof(int), s));
  GD_CUDA(ctx, cudaMemsetAsync(ctx->d_stats, 0, 32 * sizeof(unsigned long long), s));
  return GD_OK;
}

int launch_batch(gd_ctx* ctx, const DevBatch& d, cudaStream_t s, cudaEvent_t* ev, cudaStream_t s_b = nullptr,
                 cudaEvent_t mid = nullptr) {
  int launches = 0;
  DevParams pr = dev_params(ctx);
  // a field outside [0, 1] (out of the Pocket contract, scoring.hpp:15) cannot be quantised into
  // the coarse cells: the batch runs the all-FP64 kernel, reported in gd_stats.exact_fallback
  const bool field_exact = !(ctx->q_eps < 1.0f);
  if (field_exact) pr.mode = (pr.mode & ~0xff) | GD_MODE_EXACT;
  ctx->last.exact_fallback = field_exact ? 1u : 0u;
  const cudaError_t e = gdk::launch_dock(dev_pocket(ctx), pr, d, ctx->n_sms, s, &launches, ev, s_b, mid);
  ctx->last.launches = uint32_t(launches);
  if (e != cudaSuccess) return cuda_err(ctx, e, "launch_dock");
  return GD_OK;
}

// The device counters (gd_stats order) into ctx->last.
static void fill_stats(gd_ctx* ctx, const unsigned long long* st) {
  ctx->last.restarts = st[0] + st[7];  // fast sweep + restarts it handed to the FP64 kernel
  ctx->last.align_exact_evals = st[1];
  ctx->last.align_fallbacks = st[2];
  ctx->last.step_exact_evals = st[3];
  ctx->last.step_fallbacks = st[4];
  ctx->last.commits = st[5];
  ctx->last.align_second_passes = st[6];
  ctx->last.sweep_steps = st[16];
  ctx->last.sweep_invariant_steps = st[17];
  ctx->last.sweep_scored_steps = st[18];
  ctx->last.sweep_samples = st[19];
  ctx->last.cross_pairs = st[20];
  ctx->last.sweep_moves = st[21];
  ctx->last.step_exact_score_evals = st[22];
  ctx->last.step_exact_allout_evals = st[23];
  ctx->last.step_exact_face_evals = st[24];
  ctx->last.step_exact_clash_evals = st[25];
}

// name_of(l): the name of library ligand l (DegenerateAxisError names the ligand like the
// reference, molecule.cpp:156-158)
int read_device_status(gd_ctx* ctx, const std::function<std::string(uint32_t)>& name_of) {
  int err[2] = {0, 0};
  unsigned long long st[32];
  GD_CUDA(ctx, cudaMemcpy(err, ctx->d_error, sizeof err, cudaMemcpyDeviceToHost));
  GD_CUDA(ctx, cudaMemcpy(st, ctx->d_stats, sizeof st, cudaMemcpyDeviceToHost));
  fill_stats(ctx, st);
  if (err[0] == GD_ERR_DEGENERATE_AXIS) {
    return set_err(ctx, GD_ERR_DEGENERATE_AXIS, "rotamer axis atoms coincide in ligand '" + name_of(uint32_t(err[1])) + "'");
  }
  if (err[0] != 0) return set_err(ctx, err[0], "device error " + std::to_string(err[0]));
  return GD_OK;
}

// score_calls / nominal phase times are the closed form (docking.cpp:44-50, 226-229): the
// reference's recorded counters equal it by construction (docking_test.cpp:304-320).
void closed_form_counts(const gd_params& P, const gd_library* lib, uint32_t l0, uint32_t l1, gd_results* out) {
  const uint64_t G = uint64_t(P.rotation_steps[0]) * P.rotation_steps[1] * P.rotation_steps[2];
  for (uint32_t l = l0; l < l1; ++l) {
    const uint64_t R = lib->rot_off[l + 1] - lib->rot_off[l];
    const uint64_t align_calls = uint64_t(P.n_restarts) * G;
    const uint64_t opt_calls = uint64_t(P.n_restarts) * P.num_repetitions * R * P.dihedral_steps;
    if (out->score_calls) out->score_calls[l] = align_calls + opt_calls;
    if (out->phase_times) {
      out->phase_times[2 * l] = static_cast<double>(align_calls) * 1e-7;  // kNominalSecondsPerScoreCall
      out->phase_times[2 * l + 1] = static_cast<double>(opt_calls) * 1e-7;
    }
  }
}

// Result regions of a batch: (device offset, bytes, destination in out at ligand/atom/rotamer
// offsets of the chunk). Trace arrays only when requested.
struct OutCopy {
  size_t dev_off, bytes;
  void* dst;
};

std::vector<OutCopy> result_copies(const Layout& y, const gd_params& P, const gd_library* full, uint32_t l0,
                                   gd_results* out) {
  std::vector<OutCopy> v;
  const size_t a0 = full->atom_off[l0], r0 = full->rot_off[l0], N = P.n_restarts;
  v.push_back({y.o_best, y.L * sizeof(double), out->best_score + l0});
  v.push_back({y.o_brs, y.L * sizeof(uint32_t), out->best_restart + l0});
  if (out->final_xyz) v.push_back({y.o_fxyz, size_t(y.A) * 3 * sizeof(double), out->final_xyz + 3 * a0});
  if (out->final_dihedrals) v.push_back({y.o_fdih, size_t(y.Rt) * sizeof(double), out->final_dihedrals + r0});
  if (out->align_index) v.push_back({y.o_rs_aidx, y.n_items * sizeof(uint32_t), out->align_index + size_t(l0) * N});
  if (out->align_score) v.push_back({y.o_rs_ascore, y.n_items * sizeof(double), out->align_score + size_t(l0) * N});
  if (out->restart_score) v.push_back({y.o_rs_score, y.n_items * sizeof(double), out->restart_score + size_t(l0) * N});
  if (out->step_k)
    v.push_back({y.o_rs_stepk, size_t(y.Rt) * N * P.num_repetitions * sizeof(int32_t),
                 out->step_k + r0 * N * P.num_repetitions});
  return v;
}

// A library view of ligands [l0, l1) with offsets rebased to 0.
struct SubLib {
  gd_library v{};
  std::vector<uint32_t> ao, bo, ro, no;
};

void sub_library(const gd_library* lib, uint32_t l0, uint32_t l1, SubLib& s) {
  const uint32_t L = l1 - l0;
  auto rebase = [&](const uint32_t* off, std::vector<uint32_t>& o) {
    o.resize(L + 1);
    for (uint32_t i = 0; i <= L; ++i) o[i] = off[l0 + i] - off[l0];
  };
  rebase(lib->atom_off, s.ao);
  rebase(lib->bond_off, s.bo);
  rebase(lib->rot_off, s.ro);
  rebase(lib->name_off, s.no);
  s.v.n_ligands = L;
  s.v.atom_off = s.ao.data();
  s.v.xyz = lib->xyz + 3 * size_t(lib->atom_off[l0]);
  s.v.radius = lib->radius + lib->atom_off[l0];
  s.v.bond_off = s.bo.data();
  s.v.bonds = lib->bonds + 2 * size_t(lib->bond_off[l0]);
  s.v.rot_off = s.ro.data();
  s.v.rots = lib->rots + 2 * size_t(lib->rot_off[l0]);
  s.v.dihedrals = lib->dihedrals ? lib->dihedrals + lib->rot_off[l0] : nullptr;
  s.v.name_off = s.no.data();
  s.v.names = lib->names + lib->name_off[l0];
}

// Grow-only pinned / device buffers owned by the context (the executor's staging slots).
int ensure_pinned(gd_ctx* ctx, void*& p, size_t& cap, size_t need) {
  if (cap >= need) return GD_OK;
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
  GD_CUDA(ctx, cudaMallocHost(&p, need));
  cap = need;
  return GD_OK;
}

int ensure_device(gd_ctx* ctx, void*& p, size_t& cap, size_t need) {
  if (cap >= need) return GD_OK;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  GD_CUDA(ctx, cudaMalloc(&p, need));
  cap = need;
  return GD_OK;
}

}  // namespace

extern "C" {

int gd_host_pack(const gd_library* lib, const gd_params* params, const uint32_t dims[3], const double origin[3],
                 double spacing, uint32_t threads, double* seconds) {
  if (!lib || !params || !dims || !origin) return GD_ERR_ARGUMENT;
  gd_ctx tmp;  // host-only: no device state is created or touched
  tmp.params = *params;
  for (int i = 0; i < 3; ++i) {
    tmp.dims[i] = dims[i];
    tmp.origin[i] = origin[i];
  }
  tmp.spacing = spacing;
  tmp.pool = new HostPool(threads ? threads : HostPool::default_threads());
  int rc = GD_OK;
  {
    SubLib sl;
    sub_library(lib, 0, lib->n_ligands, sl);
    const Layout y = plan_layout(&sl.v, tmp.params);
    // the staging buffer is resident before the clock starts, as the executor's reused pinned
    // slots are (first-touch page faults are not packing work)
    std::vector<unsigned char> host(y.host_bytes + 256, 0);
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t bad = pack_library(&tmp, &sl.v, y, host.data());
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (bad >= 0) rc = report_invalid(&tmp, lib, uint32_t(bad));
  }
  delete tmp.pool;
  return rc;
}

int gd_stage(gd_ctx* ctx, const gd_library* lib, gd_batch** out) {
  if (!ctx || !lib || !out) return GD_ERR_ARGUMENT;
  *out = nullptr;
  if (!ctx->have_pocket) return set_err(ctx, GD_ERR_NO_POCKET, "no pocket set");
  if (!ctx->have_params) return set_err(ctx, GD_ERR_CUDA, "parameters not uploaded");
  cudaSetDevice(ctx->device);
  const uint32_t L = lib->n_ligands;
  if (L > 0 && (!lib->atom_off || !lib->bond_off || !lib->rot_off || !lib->name_off || !lib->names)) {
    return set_err(ctx, GD_ERR_ARGUMENT, "null library array");
  }
  int rc = check_contract(ctx, lib);
  if (rc != GD_OK) return rc;
  SubLib sl;
  sub_library(lib, 0, L, sl);
  auto* b = new gd_batch();
  b->ctx = ctx;
  b->params = ctx->params;
  b->n_restarts = ctx->params.n_restarts;
  b->reps = ctx->params.num_repetitions;
  b->S = ctx->params.dihedral_steps;
  b->atom_off.assign(lib->atom_off, lib->atom_off + L + 1);
  b->rot_off.assign(lib->rot_off, lib->rot_off + L + 1);
  b->name_off.assign(lib->name_off, lib->name_off + L + 1);
  if (L) b->names.assign(lib->names + lib->name_off[0], lib->name_off[L] - lib->name_off[0]);
  b->layout = plan_layout(&sl.v, ctx->params);
  const Layout& y = b->layout;
  b->arena_bytes = y.total;
  std::vector<unsigned char> host(y.host_bytes + 256);
  const int64_t bad = pack_library(ctx, &sl.v, y, host.data());  // validates every ligand first-in-order
  if (bad >= 0) {
    delete b;
    return report_invalid(ctx, lib, uint32_t(bad));
  }
  cudaError_t e = cudaMalloc(&b->arena, b->arena_bytes);
  if (e != cudaSuccess) {
    delete b;
    return cuda_err(ctx, e, "cudaMalloc(batch)");
  }
  e = cudaMemcpyAsync(b->arena, host.data(), y.host_bytes, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    cudaFree(b->arena);
    delete b;
    return cuda_err(ctx, e, "upload batch");
  }
  ctx->last.h2d_bytes = y.host_bytes;
  b->dev = bind_batch(ctx, y, static_cast<unsigned char*>(b->arena));
  *out = b;
  return GD_OK;
}

int gd_run(gd_batch* b) {
  if (!b) return GD_ERR_ARGUMENT;
  gd_ctx* ctx = b->ctx;
  cudaSetDevice(ctx->device);
  int rc = reset_device_status(ctx, ctx->stream);
  if (rc != GD_OK) return rc;
  return launch_batch(ctx, b->dev, ctx->stream, ctx->ev);
}

int gd_last_kernel_ms(gd_ctx* ctx, float* ms, uint32_t n) {
  if (!ctx || !ms) return GD_ERR_ARGUMENT;
  GD_CUDA(ctx, cudaEventSynchronize(ctx->ev[3]));
  for (uint32_t i = 0; i < n && i < 3; ++i) GD_CUDA(ctx, cudaEventElapsedTime(ms + i, ctx->ev[i], ctx->ev[i + 1]));
  return GD_OK;
}

int gd_last_run_times(gd_ctx* ctx, double* out, uint32_t n) {
  if (!ctx || !out) return GD_ERR_ARGUMENT;
  for (uint32_t i = 0; i < n && i < 4; ++i) out[i] = ctx->run_times[i];
  return GD_OK;
}

int gd_sync(gd_ctx* ctx) {
  if (!ctx) return GD_ERR_ARGUMENT;
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GD_OK;
}

int gd_fetch(gd_batch* b, gd_results* out) {
  if (!b || !out || !out->best_score || !out->best_restart) return GD_ERR_ARGUMENT;
  gd_ctx* ctx = b->ctx;
  cudaSetDevice(ctx->device);
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  int rc = read_device_status(ctx, [b](uint32_t l) {
    return l + 1 < b->name_off.size()
               ? b->names.substr(b->name_off[l] - b->name_off[0], b->name_off[l + 1] - b->name_off[l])
               : std::string();
  });
  if (rc != GD_OK) return rc;
  const Layout& y = b->layout;
  gd_library shim{};
  shim.atom_off = b->atom_off.data();
  shim.rot_off = b->rot_off.data();
  size_t d2h = 0;
  for (const OutCopy& c : result_copies(y, b->params, &shim, 0, out)) {
    GD_CUDA(ctx, cudaMemcpy(c.dst, static_cast<unsigned char*>(b->arena) + c.dev_off, c.bytes, cudaMemcpyDeviceToHost));
    d2h += c.bytes;
  }
  ctx->last.d2h_bytes = d2h;
  closed_form_counts(b->params, &shim, 0, y.L, out);
  return GD_OK;
}

int gd_topk(gd_batch* b, uint32_t k, gd_hit* out, uint32_t* n_out) {
  if (!b || !out || !n_out) return GD_ERR_ARGUMENT;
  gd_ctx* ctx = b->ctx;
  cudaSetDevice(ctx->device);
  const uint32_t n = b->dev.n_lig;
  if (k > n) k = n;
  *n_out = k;
  if (k == 0) return GD_OK;
  const size_t need = gdk::topk_scratch_bytes(n);
  if (b->topk_bytes < need) {
    cudaFree(b->topk_scratch);
    b->topk_scratch = nullptr;
    GD_CUDA(ctx, cudaMalloc(&b->topk_scratch, need));
    b->topk_bytes = need;
  }
  if (!b->d_hits) GD_CUDA(ctx, cudaMalloc(&b->d_hits, sizeof(gd_hit) * n));
  GD_CUDA(ctx, gdk::launch_topk(b->dev, k, b->topk_scratch, b->topk_bytes, b->d_hits, ctx->stream));
  GD_CUDA(ctx, cudaMemcpyAsync(out, b->d_hits, sizeof(gd_hit) * k, cudaMemcpyDeviceToHost, ctx->stream));
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GD_OK;
}

void gd_batch_free(gd_batch* b) {
  if (!b) return;
  cudaSetDevice(b->ctx->device);
  cudaFree(b->arena);
  cudaFree(b->topk_scratch);
  cudaFree(b->d_hits);
  delete b;
}

int gd_last_stats(gd_ctx* ctx, gd_stats* out) {
  if (!ctx || !out) return GD_ERR_ARGUMENT;
  // device counters of the last gd_run (synchronises the context stream)
  unsigned long long st[32];
  GD_CUDA(ctx, cudaMemcpyAsync(st, ctx->d_stats, sizeof st, cudaMemcpyDeviceToHost, ctx->stream));
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (const char* env = std::getenv("GD_PRINT_PHASES")) {
    if (env[0] == '1') {
      const char* names[8] = {"setup", "align-coarse", "align-refine", "refresh", "step-head", "step-coarse-cand",
                              "step-decide", "tail"};
      unsigned long long tot = 0;
      for (int i = 0; i < 8; ++i) tot += st[8 + i];
      for (int i = 0; i < 8; ++i) std::fprintf(stderr, "phase %-16s %6.2f%%\n", names[i], tot ? 100.0 * st[8 + i] / tot : 0.0);
    }
  }
  fill_stats(ctx, st);
  *out = ctx->last;
  return GD_OK;
}

// The executor (run_screening, pipeline.cpp:187-290, re-designed for one GPU): the library is
// cut into chunks; three staging slots (pinned host input/output + device arena + copy stream)
// rotate, so the host validates and packs chunk c+1 while the GPU runs earlier chunks. Every
// chunk's K1a runs in order on one compute stream and its K1b + K2 on a second one, so chunk c+1's
// alignment overlaps chunk c's sweep (their persistent CTAs share the SMs) and chunks complete in
// order, one at a time. H2D and D2H run on the slot's copy stream, ordered by events. Results are
// written in library order; an invalid ligand is reported before any of its chunk's work
// (earlier chunks' results are discarded with the error, as the reference's rethrow after join
// discards them, pipeline.cpp:262-272).
int gd_dock_batch(gd_ctx* ctx, const gd_library* lib, gd_results* out) {
  const double t_entry = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  if (!ctx || !lib || !out || !out->best_score || !out->best_restart) return GD_ERR_ARGUMENT;
  if (!ctx->have_pocket) return set_err(ctx, GD_ERR_NO_POCKET, "no pocket set");
  if (!ctx->have_params) return set_err(ctx, GD_ERR_CUDA, "parameters not uploaded");
  cudaSetDevice(ctx->device);
  const uint32_t L = lib->n_ligands;
  if (L > 0 && (!lib->atom_off || !lib->bond_off || !lib->rot_off || !lib->name_off || !lib->names)) {
    return set_err(ctx, GD_ERR_ARGUMENT, "null library array");
  }
  int rc = check_contract(ctx, lib);
  if (rc != GD_OK) return rc;
  const gd_params P = ctx->params;
  // Chunk schedule: a small first chunk so the GPU starts early, then each chunk 4x the previous
  // (the host packs ~7x faster than the GPU docks, so packing the next chunk stays hidden behind
  // the current one) up to kMaxChunk. Few, large launches keep the kernels' tails small.
  // GD_CHUNK=n forces uniform chunks of n ligands (experiments).
  constexpr uint32_t kMaxChunk = 16384;
  std::vector<uint32_t> bounds{0};
  {
    uint32_t fixed = 0;
    if (const char* e = std::getenv("GD_CHUNK")) fixed = std::max<uint32_t>(1, uint32_t(std::atoi(e)));
    // growth: chunk c+1 is packed while the GPU docks chunk c, so it may be at most (host packing
    // rate / GPU rate) times larger without the GPU waiting: ~0.7 per host thread of the pool
    // (~5 us per C2 ligand per thread vs ~3.7 us per ligand on the GPU), 4 at most. With few
    // threads (one rank of eight on a node) the first chunk is smaller too.
    const unsigned hw_pool = pool_of(ctx).threads();
    uint32_t next = fixed ? fixed : std::min<uint32_t>(1024, std::max<uint32_t>(hw_pool >= 8 ? 256 : 128, L / 16));
    double growth = std::min(4.0, std::max(1.5, 0.7 * double(hw_pool)));
    if (const char* e = std::getenv("GD_CHUNK0")) next = std::max<uint32_t>(1, uint32_t(std::atoi(e)));
    if (const char* e = std::getenv("GD_CHUNK_GROWTH")) growth = std::max(1.0, std::atof(e));
    while (bounds.back() < L) {
      bounds.push_back(bounds.back() + std::min(next, L - bounds.back()));
      if (!fixed) next = uint32_t(std::min<double>(kMaxChunk, std::ceil(double(next) * growth)));
    }
  }
  const uint32_t n_chunks = uint32_t(bounds.size() - 1);
  rc = reset_device_status(ctx, ctx->stream);
  if (rc != GD_OK) return rc;
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  // a slot's device arena may be reused only after the K1b that last read it: its done event
  // (D2H complete) already orders after that K1b, and drain() waits for it before reuse
  struct Pending {
    bool busy = false;
    uint32_t l0 = 0, l1 = 0;
    Layout y;
    std::vector<OutCopy> copies;
  } pend[kSlots];
  size_t h2d = 0, d2h = 0;
  // GD_TRACE_EXECUTOR=1: per-chunk host timings (validate, pack, wait for the slot) to stderr
  const bool trace = std::getenv("GD_TRACE_EXECUTOR") != nullptr;
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_start = t_entry;
  cudaStream_t sb = std::getenv("GD_ONE_STREAM") ? ctx->sa : ctx->sb;
  if (trace) std::fprintf(stderr, "executor: prologue (t=%.3f)\n", now() - t_start);
  double host_wait_ms = 0.0, align_ms = 0.0, opt_ms = 0.0;
  auto drain = [&](int si) -> int {
    Pending& p = pend[si];
    if (!p.busy) return GD_OK;
    const double tw = now();
    GD_CUDA(ctx, cudaEventSynchronize(ctx->slot[si].done));
    const double waited = now() - tw;
    host_wait_ms += waited;
    {
      float ka = 0.f, kb = 0.f;
      GD_CUDA(ctx, cudaEventElapsedTime(&ka, ctx->slot[si].a0, ctx->slot[si].mid));
      GD_CUDA(ctx, cudaEventElapsedTime(&kb, ctx->slot[si].mid, ctx->slot[si].k));
      align_ms += ka;
      opt_ms += kb;
    }
    if (trace) std::fprintf(stderr, "executor: chunk [%u,%u) wait %.3f ms\n", p.l0, p.l1, waited);
    const double t1 = trace ? now() : 0.0;
    // unpack: pinned output staging -> the caller's arrays (library order)
    const unsigned char* src = static_cast<const unsigned char*>(ctx->slot[si].h_out);
    {
      // pieces of <= 256 KB over the host pool (the caller's arrays are pageable, first touch)
      struct Piece {
        unsigned char* dst;
        const unsigned char* src;
        size_t bytes;
      };
      std::vector<Piece> pieces;
      size_t at = 0;
      for (const OutCopy& c : p.copies) {
        for (size_t o = 0; o < c.bytes; o += size_t(1) << 18)
          pieces.push_back({static_cast<unsigned char*>(c.dst) + o, src + at + o, std::min(c.bytes - o, size_t(1) << 18)});
        at += (c.bytes + 255) & ~size_t(255);
      }
      parallel_for(ctx, pieces.size(), 1, [&](size_t i) { std::memcpy(pieces[i].dst, pieces[i].src, pieces[i].bytes); });
    }
    closed_form_counts(P, lib, p.l0, p.l1, out);
    if (trace) std::fprintf(stderr, "executor: chunk [%u,%u) unpack %.3f ms\n", p.l0, p.l1, now() - t1);
    p.busy = false;
    return GD_OK;
  };
  for (uint32_t c = 0; c < n_chunks; ++c) {
    const int si = int(c % kSlots);
    auto& slot = ctx->slot[si];
    rc = drain(si);
    if (rc != GD_OK) return rc;
    const uint32_t l0 = bounds[c], l1 = bounds[c + 1];
    SubLib sl;
    sub_library(lib, l0, l1, sl);
    Pending& p = pend[si];
    p.l0 = l0;
    p.l1 = l1;
    p.y = plan_layout(&sl.v, P);
    p.copies = result_copies(p.y, P, lib, l0, out);
    size_t out_bytes = 0;
    for (const OutCopy& oc : p.copies) out_bytes += (oc.bytes + 255) & ~size_t(255);
    if ((rc = ensure_pinned(ctx, slot.h_in, slot.h_in_cap, p.y.host_bytes + 256)) != GD_OK) return rc;
    if ((rc = ensure_pinned(ctx, slot.h_out, slot.h_out_cap, out_bytes + 256)) != GD_OK) return rc;
    if ((rc = ensure_device(ctx, slot.d_arena, slot.d_cap, p.y.total)) != GD_OK) return rc;
    const double tp = trace ? now() : 0.0;
    // validation + packing in one pass; the first invalid ligand in library order is reported
    // before any of its chunk's work (earlier chunks' results are discarded with the error)
    const int64_t bad = pack_library(ctx, &sl.v, p.y, static_cast<unsigned char*>(slot.h_in));
    if (trace) std::fprintf(stderr, "executor: chunk [%u,%u) validate+pack %.3f ms (t=%.3f)\n", l0, l1, now() - tp, tp - t_start);
    if (bad >= 0) {
      cudaDeviceSynchronize();
      return report_invalid(ctx, lib, l0 + uint32_t(bad));
    }
    unsigned char* D = static_cast<unsigned char*>(slot.d_arena);
    GD_CUDA(ctx, cudaMemcpyAsync(D, slot.h_in, p.y.host_bytes, cudaMemcpyHostToDevice, slot.stream));
    GD_CUDA(ctx, cudaEventRecord(slot.in, slot.stream));
    h2d += p.y.host_bytes;
    GD_CUDA(ctx, cudaStreamWaitEvent(ctx->sa, slot.in, 0));
    if (c == 0) GD_CUDA(ctx, cudaEventRecord(ctx->run0, ctx->sa));
    GD_CUDA(ctx, cudaEventRecord(slot.a0, ctx->sa));
    rc = launch_batch(ctx, bind_batch(ctx, p.y, D, l0), ctx->sa, nullptr, sb, slot.mid);
    if (rc != GD_OK) return rc;
    GD_CUDA(ctx, cudaEventRecord(slot.k, sb));
    if (c + 1 == n_chunks) GD_CUDA(ctx, cudaEventRecord(ctx->run1, sb));
    GD_CUDA(ctx, cudaStreamWaitEvent(slot.stream, slot.k, 0));
    size_t at = 0;
    for (const OutCopy& oc : p.copies) {
      GD_CUDA(ctx, cudaMemcpyAsync(static_cast<unsigned char*>(slot.h_out) + at, D + oc.dev_off, oc.bytes,
                                   cudaMemcpyDeviceToHost, slot.stream));
      at += (oc.bytes + 255) & ~size_t(255);
      d2h += oc.bytes;
    }
    GD_CUDA(ctx, cudaEventRecord(slot.done, slot.stream));
    p.busy = true;
  }
  for (uint32_t k = 0; k < kSlots; ++k) {
    const int si = int((n_chunks + k) % kSlots);  // remaining chunks in submission order
    rc = drain(si);
    if (rc != GD_OK) return rc;
  }
  if (trace) std::fprintf(stderr, "executor: drained (t=%.3f)\n", now() - t_start);
  {
    float busy = 0.f;
    if (n_chunks) GD_CUDA(ctx, cudaEventElapsedTime(&busy, ctx->run0, ctx->run1));
    ctx->run_times[0] = 1e-3 * busy;
    ctx->run_times[1] = 1e-3 * align_ms;
    ctx->run_times[2] = 1e-3 * opt_ms;
    ctx->run_times[3] = 1e-3 * host_wait_ms;
  }
  rc = read_device_status(ctx, [lib](uint32_t l) {
    return l < lib->n_ligands ? std::string(lib->names + lib->name_off[l], lib->name_off[l + 1] - lib->name_off[l])
                              : std::string();
  });
  if (trace) std::fprintf(stderr, "executor: done (t=%.3f)\n", now() - t_start);
  ctx->last.h2d_bytes = h2d;
  ctx->last.d2h_bytes = d2h;
  return rc;
}

}  // extern "C"
