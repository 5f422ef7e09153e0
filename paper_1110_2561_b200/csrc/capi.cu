// C ABI of the B200 enumeration engine (include/isingdos_b200.h).
//
// Host-side orchestration only: argument validation, range splitting into
// run-aligned bodies and unaligned head/tail pieces, per-device cached
// streams and buffers, error strings.  All counting happens in the kernels
// of enumerate.cu / thermo.cu; there is no CPU fallback.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "isd_internal.h"

namespace isd {

static thread_local std::string g_err;
// which kernel path the last enumeration on this thread used
static thread_local std::string g_kernel_info = "none";
static std::atomic<uint64_t> g_launches{0};

uint64_t bump_launches(uint64_t n) { return g_launches += n; }

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

static int cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? ISD_ENOMEM : ISD_ECUDA,
              "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}


uint32_t hist_words_for(uint32_t nbins) { return (nbins + 31u) & ~31u; }

int hist_count_for(uint32_t hist_words) {
  // Shared-memory budget per block for the histograms.  Three 72 KB blocks
  // of 512 threads fill an SM's 228 KB.  Tunable for experiments.
  const long budget = knob_long("ISD_HIST_BYTES", 72 * 1024);
  long n = budget / (long)(hist_words * 4);
  const long cap = knob_long("ISD_NHIST_MAX", 16);
  if (n > cap) n = cap;
  if (n < 1) n = 1;
  return (int)n;
}

struct DevState {
  std::mutex mu;  // serialises host-buffer calls on this device only
  bool init = false;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  unsigned long long* d_counts = nullptr;  // (41 x 121) max table
  size_t d_counts_bytes = 0;
  double* d_buf = nullptr;  // thermo table/fields/temps/out
  size_t d_buf_bytes = 0;
  void* h_stage = nullptr;  // pinned staging for the host-buffer calls
  size_t h_stage_bytes = 0;
  // multi-device walks: the combined table (root), and local copies of
  // tables of devices this one has no peer access to
  unsigned long long* d_sum = nullptr;
  size_t d_sum_bytes = 0;
  unsigned long long* d_copies = nullptr;
  size_t d_copies_bytes = 0;
};
static DevState g_dev[64];

// (Re)allocate a device buffer of at least `bytes` on the current device.
template <class T>
static int ensure_buffer(T** ptr, size_t* have, size_t bytes,
                         const char* what) {
  if (*have >= bytes) return ISD_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) return cuda_fail(e, what);
  *have = bytes;
  return ISD_OK;
}

// Pinned host staging of at least `bytes` (grown on demand): host-buffer
// calls copy through it so their transfers are true async DMA, not the
// driver's pageable bounce path.
static int stage_buffer(DevState* s, size_t bytes, void** out) {
  if (s->h_stage_bytes < bytes) {
    if (s->h_stage) cudaFreeHost(s->h_stage);
    s->h_stage = nullptr;
    s->h_stage_bytes = 0;
    const size_t want = bytes < 65536 ? 65536 : bytes;
    cudaError_t e = cudaHostAlloc(&s->h_stage, want, cudaHostAllocDefault);
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc(staging)");
    s->h_stage_bytes = want;
  }
  *out = s->h_stage;
  return ISD_OK;
}

// Select `device` on this thread, initialise its state once, and lock it:
// host-buffer calls on different devices run concurrently (one host thread
// per GPU in full_dos_timed), calls on one device are serialised.
static int get_dev(int device, DevState** out,
                   std::unique_lock<std::mutex>* lock) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(ISD_ENODEV, "no CUDA device available (%s)",
                e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  if (device < 0 || device >= ndev || device >= 64)
    return fail(ISD_ENODEV, "device %d outside [0, %d)", device, ndev);
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  DevState& s = g_dev[device];
  *lock = std::unique_lock<std::mutex>(s.mu);
  if (!s.init) {
    e = cudaDeviceGetAttribute(&s.sm_count, cudaDevAttrMultiProcessorCount,
                               device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
    cudaEventCreate(&s.ev0);
    cudaEventCreate(&s.ev1);
    s.init = true;
  }
  *out = &s;
  return ISD_OK;
}

// SMs the enumeration grids are sized for: the device's, or fewer under the
// ISD_GRID_SMS test knob (which stands in for a small partition of a GPU,
// e.g. a MIG slice or a green context).
static int current_sm_count(int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  e = cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  const long cap = knob_long("ISD_GRID_SMS", 0);
  if (cap > 0 && cap < *sms) *sms = (int)cap;
  return ISD_OK;
}

// Configurations per launch.  Every grid has at least one block per SM and
// a block's u32 shared counters see at most the configurations its block
// counts (one RED lane adds 1 for 1, 2 or 4 configurations), so with
// launches of at most 2^31 configurations per SM of the grid no counter can
// wrap, even for a work item twice the mean (banded launches cut one item
// per block, of equal modelled cost).  A power of two, so that a banded
// launch chunk stays an aligned power-of-two range.  148 SMs: 2^38.
static uint64_t launch_cap(int sms) {
  uint64_t p = 1;
  while (p * 2 <= (uint64_t)(sms < 1 ? 1 : sms)) p *= 2;
  return p << 31;
}

// Restores the calling thread's current device on scope exit.  The library
// shares the primary context with its caller (e.g. torch); a call on device
// k must not leave the caller's thread switched to k.
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      cudaGetLastError();
    }
  }
  ~DeviceGuard() {
    int now = -1;
    if (prev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != prev)
      cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Plans are compiled once per (lattice, loop width): the layout search
// replays a sample of warp instructions and costs tens of milliseconds.
// The model ranks every layout; before the first walk of >= 2^33
// configurations the best 40 are timed on the GPU on a 2^33-configuration
// sample of warps spread over the range, and the best 6 of those on a
// contiguous slice of up to 2^36 configurations; the fastest is kept
// (autotune, once per process, lattice and loop width; ISD_AUTOTUNE=0
// disables).
struct PlanEntry {
  int rc = 0;
  isd_plan_info info;
  std::vector<isd_plan_info> ranked;
  bool tuned = false;
};
static std::mutex g_plan_mu;
static std::map<std::string, PlanEntry> g_plans;

// top: the configuration bits a walk holds fixed (a shard of an aligned
// power-of-two split: its start), which the layout model includes
static std::string plan_key(const isd_lattice* lat, uint64_t hint,
                            uint64_t top = 0) {
  const int l = plan_loop_bits(lat, hint);
  std::string key(reinterpret_cast<const char*>(lat), sizeof(*lat));
  key.push_back((char)l);
  key += "|top" + std::to_string(top);
  key += knob_signature();
  return key;
}

static int cached_plan(const isd_lattice* lat, uint64_t hint,
                       isd_plan_info* info, uint64_t top = 0) {
  const std::string key = plan_key(lat, hint, top);
  std::lock_guard<std::mutex> lock(g_plan_mu);
  auto it = g_plans.find(key);
  if (it == g_plans.end()) {
    NvtxRange nvtx("isd:plan model");
    PlanEntry fresh;
    fresh.rc = compile_plan(lat, hint, &fresh.info, &fresh.ranked, top);
    it = g_plans.emplace(key, std::move(fresh)).first;
  }
  *info = it->second.info;
  return it->second.rc;
}

// ---- banded launches ------------------------------------------------------
// A banded plan needs an aligned power-of-two run range: its work items
// cover the free run bits in popcount order.
static int log2_exact(uint64_t x) {
  return (x && !(x & (x - 1))) ? 63 - __builtin_clzll(x) : -1;
}

static bool band_ok(const isd_plan_info& info, uint64_t start, uint64_t end) {
  if (!info.band_rows) return false;
  const uint64_t unit = 1ull << info.k;
  if (start % unit || end % unit || end <= start) return false;
  const int rb = log2_exact((end - start) >> info.k);
  uint64_t span_bits = info.lane_mask;
  for (int v = 0; v < 5; ++v) span_bits |= info.lane_vec[v];
  return rb >= 6 && lane_span(span_bits) <= rb;
}

static std::mutex g_items_mu;
struct ItemSet {
  BandItem* dev = nullptr;
  uint32_t count = 0;
  std::vector<BandItem> host;
};
static std::map<std::string, ItemSet> g_items;

// Device work items for 2^F slots (uploaded once per device, size and cost
// curve; `cost_key` identifies w).
// Cost curves of a banded launch per segment of its slot order: rows
// ascending, rows descending (a mirrored item), and the cheaper of the two
// (ISD_BAND_MIRROR: 0 = never mirror, 1 = per item, 2 = always).
struct CostCurves {
  std::vector<double> fwd, mir, best;
  std::string name;  // short name of `best` for the items cache
  uint8_t pos[24];   // slot bit i -> run bit (band_slot_order)
  std::string disk_key;  // of the "cost3" cache entry
  long mirror_mode = 1;
  int calibrated = 0;    // rounds of measured correction applied
};

// `best`, and the curves' short name, from fwd / mir
static void finish_curves(CostCurves* cc) {
  cc->best.resize(cc->fwd.size());
  for (size_t i = 0; i < cc->fwd.size(); ++i)
    cc->best[i] = cc->mirror_mode == 0   ? cc->fwd[i]
                  : cc->mirror_mode == 2 ? cc->mir[i]
                                         : std::min(cc->fwd[i], cc->mir[i]);
  // the items cache names the curves by a hash of their rounded values
  uint64_t h = 1469598103934665603ull;
  for (const std::vector<double>* v : {&cc->best, &cc->fwd, &cc->mir})
    for (double x : *v) {
      h ^= (uint64_t)std::llround(x * 1e4);
      h *= 1099511628211ull;
    }
  for (uint8_t b : cc->pos) {
    h ^= b;
    h *= 1099511628211ull;
  }
  cc->name = "w" + std::to_string(h) + ":" + std::to_string(cc->best.size());
}

static std::string curves_blob(const CostCurves& cc) {
  std::string put(reinterpret_cast<const char*>(cc.fwd.data()),
                  cc.fwd.size() * sizeof(double));
  put.append(reinterpret_cast<const char*>(cc.mir.data()),
             cc.mir.size() * sizeof(double));
  put.append(reinterpret_cast<const char*>(cc.pos), sizeof cc.pos);
  return put;
}

static int band_items(int F, int n_target, int span, const CostCurves* cc,
                      double flush_units, BandItem** ptr, uint32_t* count,
                      std::vector<BandItem>* host_out = nullptr) {
  static const std::vector<double> equal;
  const std::vector<double>& w = cc ? cc->best : equal;
  const long mirror_mode = knob_long("ISD_BAND_MIRROR", 1);
  const std::string cost_key =
      (cc ? cc->name : std::string()) + ":m" + std::to_string(mirror_mode);
  int dev = 0;
  cudaGetDevice(&dev);
  const std::string key = std::to_string(dev) + ":" + std::to_string(F) +
                          ":" + std::to_string(n_target) + ":" +
                          std::to_string(span) + ":" + cost_key + ":" +
                          std::to_string((int)flush_units);
  std::lock_guard<std::mutex> lock(g_items_mu);
  auto it = g_items.find(key);
  if (it == g_items.end()) {
    // the kernel's register unrank is exact in u32 up to F = 23
    if (F > 23) return fail(ISD_EINVAL, "banded launch: too many slot bits");
    // the class-boundary cuts add a few small items: shrink the target so
    // the count stays a whole number of waves (blocks get equal work)
    // (exact: n_target items, block b walks item b, plus the small items
    // of the extreme classes as second items of blocks 0 and 1; otherwise
    // the target is shrunk until the count is a whole number of waves)
    auto cut_items = [&](const std::vector<double>& curve) {
      bool exact = false;
      std::vector<BandItem> items =
          band_work_items(F, n_target, span, curve, flush_units, &exact);
      for (int goal = n_target;
           !exact && (int)items.size() > n_target && goal > 1;) {
        goal -= (int)items.size() - n_target;
        bool ignored = false;
        items = band_work_items(F, goal < 1 ? 1 : goal, span, curve,
                                flush_units, &ignored);
      }
      return items;
    };
    // an item's table holds its rows in descending order where that costs
    // fewer wavefronts over the item's slots
    const bool per_item = mirror_mode == 1 && cc && !cc->mir.empty();
    auto mark = [&](std::vector<BandItem>* items) {
      const uint64_t total = 1ull << F, n_seg = cc ? cc->fwd.size() : 1;
      for (BandItem& x : *items) {
        x.mirror = mirror_mode == 2 ? 1u : 0u;
        if (!per_item) continue;
        double cf = 0, cm = 0;
        for (uint64_t j = x.g0 * n_seg / total;
             j < n_seg && total * j / n_seg < x.g1; ++j) {
          const uint64_t lo = std::max<uint64_t>(x.g0, total * j / n_seg);
          const uint64_t hi = std::min<uint64_t>(x.g1, total * (j + 1) / n_seg);
          if (hi > lo) {
            cf += (double)(hi - lo) * cc->fwd[j];
            cm += (double)(hi - lo) * cc->mir[j];
          }
        }
        x.mirror = cm < cf ? 1u : 0u;
      }
    };
    std::vector<BandItem> host = cut_items(w);
    mark(&host);
    // One order of rows serves a whole item, so an item costs the smaller
    // of its two sums, not the sum of its segments' smaller costs: re-cut
    // on the curve the items' own choices make (a segment costs what the
    // item holding its first slot chose) until the choices settle.
    for (int round = 0; per_item && round < 4; ++round) {
      const uint64_t total = 1ull << F, n_seg = cc->fwd.size();
      std::vector<BandItem> by_start(host);
      std::sort(by_start.begin(), by_start.end(),
                [](const BandItem& a, const BandItem& b) { return a.g0 < b.g0; });
      std::vector<double> eff(n_seg);
      size_t k = 0;
      for (uint64_t j = 0; j < n_seg; ++j) {
        const uint64_t lo = total * j / n_seg;
        while (k + 1 < by_start.size() && by_start[k].g1 <= lo) ++k;
        eff[j] = by_start[k].mirror ? cc->mir[j] : cc->fwd[j];
      }
      std::vector<BandItem> next = cut_items(eff);
      mark(&next);
      bool same = next.size() == host.size();
      for (size_t i = 0; same && i < next.size(); ++i)
        same = next[i].g0 == host[i].g0 && next[i].g1 == host[i].g1 &&
               next[i].mirror == host[i].mirror;
      host.swap(next);
      if (same) break;
    }
    // the items must tile [0, 2^F) (listed in any order), each within
    // span + 1 popcount classes of its q0
    {
      std::vector<BandItem> r(host);
      std::sort(r.begin(), r.end(), [](const BandItem& a, const BandItem& b) {
        return a.g0 < b.g0;
      });
      std::vector<uint64_t> cum(F + 2, 0);
      uint64_t c = 1;
      for (int q = 0; q <= F; ++q) {
        cum[q + 1] = cum[q] + c;
        c = c * (uint64_t)(F - q) / (uint64_t)(q + 1);
      }
      auto cls = [&](uint64_t g) {
        int q = 0;
        while (cum[q + 1] <= g) ++q;
        return q;
      };
      uint64_t next = 0;
      for (const BandItem& x : r) {
        if (x.g0 != next || x.g1 <= x.g0 || cls(x.g0) != (int)x.q0 ||
            cls(x.g1 - 1) > (int)x.q0 + span)
          return fail(ISD_EINVAL, "band work items do not tile the slots");
        next = x.g1;
      }
      if (next != (1ull << F))
        return fail(ISD_EINVAL, "band work items do not tile the slots");
    }
    const size_t item_bytes = host.size() * sizeof(BandItem);
    BandItem* d = nullptr;
    // (the caller's stream may be capturing a graph: this upload is not part
    // of the captured work, so this thread steps out of the capture rules)
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    cudaError_t e = cudaMalloc(&d, item_bytes);
    cudaStream_t up = nullptr;  // not the legacy stream: it joins blocking ones
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d, host.data(), item_bytes, cudaMemcpyHostToDevice, up);
    if (e == cudaSuccess) e = cudaStreamSynchronize(up);
    if (up) cudaStreamDestroy(up);
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (e != cudaSuccess) return cuda_fail(e, "band work items");
    ItemSet set;
    set.dev = d;
    set.count = (uint32_t)host.size();
    set.host = host;
    it = g_items.emplace(key, std::move(set)).first;
  }
  *ptr = it->second.dev;
  *count = it->second.count;
  if (host_out) *host_out = it->second.host;
  return ISD_OK;
}

// Cost curves of a banded launch (cached: same lattice, plan, lanes and run
// base give the same curves).  ISD_BAND_WEIGHTS=0: equal costs.
static std::mutex g_cost_mu;
static std::map<std::string, CostCurves> g_cost;

static void band_costs(const isd_lattice* lat, const isd_plan_info& info,
                       const HoistParams& hp, int run_bits,
                       const CostCurves** out) {
  *out = nullptr;
  if (knob_long("ISD_BAND_WEIGHTS", 1) == 0) return;
  const long mirror_mode = knob_long("ISD_BAND_MIRROR", 1);
  // (explicit fields: the structs' padding is not initialised)
  std::string k;
  auto add = [&](unsigned long long v) { k += std::to_string(v) + ","; };
  add(lat->n_spins);
  for (uint32_t c = 0; c < lat->n_classes; ++c) {
    add(lat->classes[c].shift);
    add(lat->classes[c].bond_mask);
    add(lat->classes[c].jneg_mask);
  }
  add(info.k);
  add(info.loop_mask);
  add(info.e_mode);
  add(info.row_words);
  add(info.e_words);
  add(info.plane_words);
  for (int i = 0; i < 2; ++i) {
    add(info.pair_words[i]);
    add(info.pair_degree[i]);
  }
  add(info.pair_mode);
  add((unsigned long long)(long long)info.pair_both);
  for (int t = 0; t < kCopyBits; ++t) add(info.copy_site[t]);
  add(hp.lane_mask);
  for (int v = 0; v < 5; ++v) add(hp.lane_vec[v]);
  add(hp.run_begin);
  add((unsigned long long)run_bits);
  // slots ordered by the run sites that decide the items' row order
  // (ISD_BAND_ORDER=0: natural order); only with per-item mirroring
  const bool reorder = mirror_mode == 1 && knob_long("ISD_BAND_ORDER", 1) != 0;
  k += reorder ? "o1," : "o0,";
  const std::string mem_key = k + "m" + std::to_string(mirror_mode);
  {
    std::lock_guard<std::mutex> lock(g_cost_mu);
    auto it = g_cost.find(mem_key);
    if (it == g_cost.end()) {
      CostCurves cc;
      // ~16 segments per item of a four-items-per-block launch, 64
      // samples each (c5: ~0.3 s once per process and plan; then from the
      // disk cache, both curves in one entry)
      const int F = run_bits - 5;
      const int n_seg = (int)std::min<uint64_t>(1ull << F, 16ull * 4 * 148);
      std::string blob;
      std::memset(cc.pos, 0, sizeof cc.pos);
      if (cache_get("cost3", k, &blob) && blob.size() > sizeof cc.pos &&
          (blob.size() - sizeof cc.pos) % (2 * sizeof(double)) == 0) {
        const size_t n = (blob.size() - sizeof cc.pos) / (2 * sizeof(double));
        cc.fwd.resize(n);
        cc.mir.resize(n);
        std::memcpy(cc.fwd.data(), blob.data(), n * sizeof(double));
        std::memcpy(cc.mir.data(), blob.data() + n * sizeof(double),
                    n * sizeof(double));
        std::memcpy(cc.pos, blob.data() + 2 * n * sizeof(double),
                    sizeof cc.pos);
      } else {
        band_slot_order(lat, info, hp.run_begin, hp.lane_mask, hp.lane_vec,
                        run_bits, reorder, cc.pos);
        band_slot_cost(lat, info, hp.run_begin, hp.lane_mask, hp.lane_vec,
                       run_bits, n_seg, 64, &cc.fwd, &cc.mir, cc.pos);
        cache_put("cost3", k, curves_blob(cc));
      }
      cc.disk_key = k;
      cc.mirror_mode = mirror_mode;
      finish_curves(&cc);
      it = g_cost.emplace(mem_key, std::move(cc)).first;
    }
    *out = &it->second;  // (map nodes are stable)
  }
}

// Per-device ring of item-claim counters: each banded launch takes the next
// slot and zeroes it on its own stream first, so launches in flight on
// different streams never share a counter (64 slots).
static std::mutex g_claim_mu;
static std::map<int, uint32_t*> g_claim_ring;
static std::atomic<uint32_t> g_claim_next{0};
constexpr uint32_t kClaimSlots = 64;

static int claim_counter(uint32_t** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  uint32_t* ring = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_claim_mu);
    auto it = g_claim_ring.find(dev);
    if (it == g_claim_ring.end()) {
      cudaError_t e = cudaMalloc(&ring, kClaimSlots * 32);  // 32 B apart
      if (e != cudaSuccess) return cuda_fail(e, "band claim counters");
      it = g_claim_ring.emplace(dev, ring).first;
    }
    ring = it->second;
  }
  // (the launch zeroes it on its own stream first)
  *out = ring + 8 * (g_claim_next.fetch_add(1) % kClaimSlots);
  return ISD_OK;
}

// Fill the banded-launch fields of hp for its run range [run_begin, run_end)
// (a dynamic-claim counter must be zeroed on the launch's stream first).
static int set_band_launch(const isd_lattice* lat, const isd_plan_info& info,
                           HoistParams* hp, int sms, bool weighted = true,
                           const CostCurves** cc_out = nullptr,
                           std::vector<BandItem>* host_out = nullptr) {
  hp->band_free_bits = 0;
  hp->band_items = 0;
  hp->band_n_items = 0;
  hp->band_claim = 0;
  hp->band_clk = 0;
  if (cc_out) *cc_out = nullptr;
  if (!hp->band_rows) return ISD_OK;
  const int rb = log2_exact(hp->run_end - hp->run_begin);
  if (rb < 6) return fail(ISD_EINVAL, "banded launch needs 2^r runs");
  BandItem* items = nullptr;
  uint32_t count = 0;
  // One item per block: items are cut to equal modelled cost
  // (band_slot_cost), so blocks finish together without the extra flushes
  // of several items per block.  Measured on c5: 2^36 walk 2.253 ms with
  // four equal-size items per block -> 2.201 ms with one cost-weighted
  // item; 2^33 shards 0.33-0.38 -> 0.30-0.33 ms.  Without weights
  // (ISD_BAND_WEIGHTS=0) up to four items per block of >= 512 slots mix
  // popcount classes instead.
  const int F = rb - 5;
  long dflt = (long)((1ull << F) / (512ull * (uint64_t)sms));
  dflt = dflt < 1 ? 1 : (dflt > 4 ? 4 : dflt);
  if (weighted && knob_long("ISD_BAND_WEIGHTS", 1) != 0) dflt = 1;
  const int per_sm = (int)knob_long("ISD_BAND_ITEMS_PER_SM", dflt);
  const CostCurves* cc = nullptr;
  if (weighted) band_costs(lat, info, *hp, rb, &cc);
  // a flush (~20 K SM cycles) in units of one slot's walk at one wavefront
  // per RED (a slot = 32 lanes x 2^l loop subsets x 32 REDs / 32 lanes)
  const double flush_units =
      20000.0 / (double)((hp->pair == 3 ? 16u : 32u) << hp->l);
  const int rc = band_items(F, (per_sm < 1 ? 1 : per_sm) * sms,
                            (int)hp->band_span, cc, flush_units, &items,
                            &count, host_out);
  if (rc) return rc;
  if (cc_out) *cc_out = cc;
  hp->band_free_bits = (uint32_t)(rb - 5);
  // the slot map: the cost model's order, else the natural one
  {
    uint8_t natural[24];
    const uint8_t* pos = cc ? cc->pos : natural;
    if (!cc)
      band_slot_order(lat, info, hp->run_begin, hp->lane_mask, hp->lane_vec,
                      rb, false, natural);
    if (band_slot_fields(pos, rb - 5, hp->slot_mask, hp->slot_rot) < 0)
      return fail(ISD_EINVAL, "banded launch: slot map needs too many fields");
  }
  hp->band_items = (uint64_t)(uintptr_t)items;
  hp->band_n_items = count;
  // ISD_BAND_DYNAMIC=1: blocks claim items from a counter (measured no
  // faster than the static round-robin over items in slot order)
  if (knob_long("ISD_BAND_DYNAMIC", 0) != 0) {
    uint32_t* slot = nullptr;
    const int rc2 = claim_counter(&slot);
    if (rc2) return rc2;
    hp->band_claim = (uint64_t)(uintptr_t)slot;
  }
  return ISD_OK;
}

// Correct a banded launch's cost curves by measurement.  The model scores a
// slot by its expected wavefronts; what a block spends on an item also
// holds issue-bound stretches and the flush, and the model's estimate of
// the mirrored order is a few percent off in the upper popcount classes
// (c5: block totals within -1.5%/+2.5% of their mean).  One launch over the
// walk's own range writes every item's SM cycles (k1_body.cuh item_clk);
// each segment's costs are scaled by measured / modelled of the item that
// held it, the items are cut again, and a second round settles what the
// moved boundaries changed.  The corrected curves replace the model's in
// memory and in the disk cache (the plan is tuned once per cache, so they
// are what later processes cut their items from).
static void calibrate_items(const isd_lattice* lat, const isd_plan_info& info,
                            HoistParams hp, int sms, unsigned long long* scratch,
                            cudaStream_t st, bool jit_ok) {
  if (!hp.band_rows || knob_long("ISD_BAND_CALIBRATE", 1) == 0 ||
      knob_long("ISD_BAND_WEIGHTS", 1) == 0 ||
      knob_long("ISD_BAND_DYNAMIC", 0) != 0)
    return;
  NvtxRange nvtx("isd:calibrate items");
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    if (e0) cudaEventDestroy(e0);
    cudaGetLastError();
    return;
  }
  auto launch = [&](const HoistParams& p) {
    int x = 0;
    if (jit_ok) x = launch_hoisted_jit(p, scratch, sms, st, nullptr);
    if (x <= 0) x = launch_hoisted(p, scratch, sms, st);
    if (x > 0) bump_launches(1);
    return x > 0;
  };
  // the walk's time with the current curves' items (best of three launches)
  auto walk_ms = [&](const CostCurves** cc, std::vector<BandItem>* items) {
    if (set_band_launch(lat, info, &hp, sms, true, cc, items) || !*cc ||
        items->empty() || (*cc)->fwd.empty())
      return -1.f;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      float t = 0.f;
      cudaEventRecord(e0, st);
      const bool ok = launch(hp);
      cudaEventRecord(e1, st);
      if (!ok || cudaEventSynchronize(e1) != cudaSuccess ||
          cudaEventElapsedTime(&t, e0, e1) != cudaSuccess) {
        cudaGetLastError();
        return -1.f;
      }
      best = std::min(best, t);
    }
    return best;
  };
  const CostCurves* cc = nullptr;
  std::vector<BandItem> items;
  float best_ms = walk_ms(&cc, &items);
  // The correction is kept only while the walk it yields measures faster:
  // cycles read while another process shares the GPU would otherwise go
  // into the disk cache as a lopsided cut.
  std::vector<double> keep_fwd, keep_mir;
  if (best_ms > 0) {
    keep_fwd = cc->fwd;
    keep_mir = cc->mir;
  }
  bool improved = false;
  for (int round = 0; round < 2 && best_ms > 0; ++round) {
    unsigned long long* clk = nullptr;
    const size_t bytes = items.size() * sizeof(unsigned long long);
    if (cudaMalloc(&clk, bytes) != cudaSuccess) {
      cudaGetLastError();
      break;
    }
    cudaMemsetAsync(clk, 0, bytes, st);
    hp.band_clk = (uint64_t)(uintptr_t)clk;
    const bool ok = launch(hp);
    std::vector<unsigned long long> got(items.size(), 0);
    cudaError_t e = ok ? cudaMemcpyAsync(got.data(), clk, bytes,
                                         cudaMemcpyDeviceToHost, st)
                       : cudaErrorUnknown;
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(clk);
    hp.band_clk = 0;
    if (e != cudaSuccess) {
      cudaGetLastError();
      break;
    }
    // modelled cost of every item in the order it chose
    const uint64_t total = 1ull << hp.band_free_bits;
    const uint64_t n_seg = cc->fwd.size();
    std::vector<double> pred(items.size(), 0.0);
    double sum_pred = 0, sum_meas = 0, slots_main = 0;
    size_t n_main = 0;
    for (const BandItem& it : items) slots_main += (double)(it.g1 - it.g0);
    slots_main /= (double)items.size();
    auto main_item = [&](size_t i) {
      // (the small items of the extreme classes carry mostly fixed costs)
      return (double)(items[i].g1 - items[i].g0) >= 0.5 * slots_main &&
             got[i] != 0;
    };
    for (size_t i = 0; i < items.size(); ++i) {
      const BandItem& it = items[i];
      const std::vector<double>& w = it.mirror ? cc->mir : cc->fwd;
      for (uint64_t j = it.g0 * n_seg / total;
           j < n_seg && total * j / n_seg < it.g1; ++j) {
        const uint64_t lo = std::max<uint64_t>(it.g0, total * j / n_seg);
        const uint64_t hi = std::min<uint64_t>(it.g1, total * (j + 1) / n_seg);
        if (hi > lo) pred[i] += (double)(hi - lo) * w[j];
      }
      if (!main_item(i)) continue;
      sum_pred += pred[i];
      sum_meas += (double)got[i];
      ++n_main;
    }
    if (n_main < 8 || sum_pred <= 0 || sum_meas <= 0) break;
    std::vector<double> ratio(items.size(), 1.0);
    bool sane = true;
    for (size_t i = 0; i < items.size(); ++i) {
      if (!main_item(i)) continue;
      const double r = ((double)got[i] / sum_meas) / (pred[i] / sum_pred);
      // (the model is good to a few percent: anything further off is a
      // disturbed measurement, not a correction)
      sane = sane && r > 0.85 && r < 1.18;
      ratio[i] = std::min(1.08, std::max(0.93, r));
    }
    if (!sane) break;
    // scale each segment by the item that held its first slot
    std::vector<size_t> order(items.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
      return items[a].g0 < items[b].g0;
    });
    {
      std::lock_guard<std::mutex> lock(g_cost_mu);
      CostCurves* mut = const_cast<CostCurves*>(cc);
      size_t kk = 0;
      for (uint64_t j = 0; j < n_seg; ++j) {
        const uint64_t lo = total * j / n_seg;
        while (kk + 1 < order.size() && items[order[kk]].g1 <= lo) ++kk;
        mut->fwd[j] *= ratio[order[kk]];
        mut->mir[j] *= ratio[order[kk]];
      }
      finish_curves(mut);
    }
    // (the second round starts from the first's cut either way; whichever
    // of the three cuts measured fastest is restored below)
    const float ms = walk_ms(&cc, &items);
    if (ms <= 0) break;
    if (ms < best_ms * 0.999f) {
      best_ms = ms;
      keep_fwd = cc->fwd;
      keep_mir = cc->mir;
      improved = true;
    }
  }
  if (cc && !keep_fwd.empty()) {
    std::lock_guard<std::mutex> lock(g_cost_mu);
    CostCurves* mut = const_cast<CostCurves*>(cc);
    mut->fwd = keep_fwd;
    mut->mir = keep_mir;
    if (improved) mut->calibrated += 1;
    finish_curves(mut);
    if (improved) cache_put("cost3", mut->disk_key, curves_blob(*mut));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

static constexpr int kTuneCandidates = 40;
static constexpr uint64_t kTuneConfigs = 1ull << 33;
static constexpr size_t kTuneFinalists = 6;
static constexpr uint64_t kTuneSliceConfigs = 1ull << 36;

// Time the model's best layouts on `st` and keep the fastest.  Synchronous.
// Candidates may differ in loop width (banded plans use a shorter loop), so
// each is timed on its own run range of [start, end).
// Returns false when the winner's two timed launches disagreed by more than
// 15% (another process was using the GPU): the pick then serves this
// process but is not written to the disk cache.
static bool autotune(const isd_lattice* lat, uint64_t hint, uint64_t start,
                     uint64_t end, int sms, isd_plan_info* info,
                     uint64_t top) {
  NvtxRange nvtx("isd:autotune");
  if (knob_long("ISD_AUTOTUNE", 1) == 0) return true;
  const std::string key = plan_key(lat, hint, top);
  std::vector<isd_plan_info> cands;
  {
    std::lock_guard<std::mutex> lock(g_plan_mu);
    PlanEntry& pe = g_plans[key];
    if (pe.tuned || pe.rc) {
      *info = pe.info;
      return true;
    }
    pe.tuned = true;
    const int n_cand = (int)knob_long("ISD_TUNE_CANDIDATES", kTuneCandidates);
    for (size_t i = 0; i < pe.ranked.size() && (int)cands.size() < n_cand;
         ++i)
      if (!pe.ranked[i].band_rows || band_ok(pe.ranked[i], start, end))
        cands.push_back(pe.ranked[i]);
  }
  if (cands.size() < 2) return true;
  // tuning runs on a private stream (never the caller's, which may be
  // capturing a graph or carry unrelated work); it is synchronous, and
  // waits for the device to drain first: a candidate timed while other
  // work still occupies the SMs would look slower than it is
  cudaDeviceSynchronize();
  cudaGetLastError();
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  const size_t bytes =
      (size_t)(lat->n_spins + 1) * (lat->n_bonds + 1) * sizeof(uint64_t);
  unsigned long long* scratch = nullptr;
  if (cudaMalloc(&scratch, bytes) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamDestroy(st);
    return true;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // run range [r0, r1) of [start, end) for a loop width of k bits
  auto run_range = [&](uint32_t k, uint64_t* r0, uint64_t* r1) {
    *r0 = (start + ((1ull << k) - 1)) >> k;
    *r1 = end >> k;
  };
  // Stage 1 (unbanded candidates): per-run ms on a sample of warps spread
  // evenly over the body, each warp with the candidate's own lane
  // placement, so every region of the index space votes and all
  // candidates see the same spread (< 0: not applicable)
  auto time_spread = [&](const isd_plan_info& cand) -> float {
    HoistParams hp;
    fill_hoist(lat, &cand, &hp);
    uint64_t run0, run1;
    run_range(cand.k, &run0, &run1);
    const uint64_t body = run1 > run0 ? run1 - run0 : 0;
    const uint64_t runs = kTuneConfigs >> cand.k;
    uint64_t span_bits = hp.lane_mask;
    for (int v = 0; v < 5; ++v) span_bits |= hp.lane_vec[v];
    const uint64_t blk = 1ull << lane_span(span_bits);
    if (body < blk || body < runs) return -1.f;
    const uint64_t warps = runs / 32;
    // warp slots must stay inside whole lane blocks of the body
    const uint64_t usable = (body / blk) * (blk / 32);
    // odd stride: a power-of-two stride would pin the low run bits of every
    // sampled warp to zero and bias the sample
    hp.hi_step = usable / warps;
    if (hp.hi_step > 1 && !(hp.hi_step & 1)) hp.hi_step -= 1;
    if (hp.hi_step < 1) hp.hi_step = 1;
    hp.run_begin = run0;
    hp.run_end = run0 + warps * 32;
    float ms = 0.f;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, st);
      launch_hoisted(hp, scratch, sms, st);
      cudaEventRecord(e1, st);
    }
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    bump_launches(2);
    return ms / (float)(warps * 32) / (float)(1ull << cand.k);  // per config
  };
  std::vector<std::pair<float, size_t>> stage1;
  std::vector<size_t> banded;
  for (size_t i = 0; i < cands.size(); ++i) {
    if (cands[i].band_rows) {
      banded.push_back(i);  // needs whole work items: straight to stage 2
      continue;
    }
    const float t = time_spread(cands[i]);
    if (t >= 0.f) stage1.push_back({t, i});
  }
  std::sort(stage1.begin(), stage1.end());
  // optional GPU hill climb of the best candidate's lane pattern, scored on
  // the same spread sample (ISD_GPU_CLIMB = steps); the result joins the
  // finalists
  const long climb = knob_long("ISD_GPU_CLIMB", 0);
  if (climb > 0 && !stage1.empty()) {
    isd_plan_info cur = cands[stage1[0].second];
    float cur_t = stage1[0].first;
    uint64_t run0, run1;
    run_range(cur.k, &run0, &run1);
    int run_bits = 0;
    while (run_bits < 63 && (2ull << run_bits) <= run1 - run0) ++run_bits;
    uint64_t seed = 0x6A09E667F3BCC909ull;
    for (long step = 0; step < climb; ++step) {
      isd_plan_info q = cur;
      if (!mutate_lanes(lat, run_bits, &seed, &q)) continue;
      const float t = time_spread(q);
      if (t >= 0.f && t < cur_t * 0.999f) {
        cur = q;
        cur_t = t;
      }
    }
    cands.push_back(cur);
    stage1.insert(stage1.begin(), {cur_t, cands.size() - 1});
  }
  // stage 2: the best few, timed as a real walk — one contiguous slice of
  // up to 2^36 configurations (the spread sample ranks the candidates but
  // not reliably enough to pick one), with the kernel the walk will use:
  // the NVRTC build when it is available (its Gray-order loop changes the
  // instruction mix), compiled once per finalist and cached for the walk.
  // The model's best banded candidates join the finalists.
  const bool jit_ok = knob_long("ISD_JIT", 1) != 0;
  std::vector<size_t> finalists;
  const size_t n_final = (size_t)knob_long("ISD_TUNE_FINALISTS", kTuneFinalists);
  // (stage 1 ran the ahead-of-time kernel, whose plain loop is issue-bound
  // in the modes with few REDs per loop subset: it ranks layouts within a
  // pairing mode, not the modes against each other, and its order within
  // the top mode is only a hint for the Gray-walking kernel — the best four
  // of the highest mode present go through, two of the next, one of each
  // other, then the best of the rest)
  {
    int top_mode = -1, next_mode = -1;
    for (const auto& s1 : stage1) {
      const int pm = (int)(cands[s1.second].pair_mode & 3u);
      if (pm > top_mode) {
        next_mode = top_mode;
        top_mode = pm;
      } else if (pm != top_mode && pm > next_mode) {
        next_mode = pm;
      }
    }
    int per_mode[4] = {0, 0, 0, 0};
    std::vector<char> taken(stage1.size(), 0);
    for (size_t s2 = 0; s2 < stage1.size(); ++s2) {
      const int pm = (int)(cands[stage1[s2].second].pair_mode & 3u);
      const int quota = pm == top_mode ? 4 : (pm == next_mode ? 2 : 1);
      if (n_final >= 4 && per_mode[pm] < quota) {
        ++per_mode[pm];
        taken[s2] = 1;
        finalists.push_back(stage1[s2].second);
      }
    }
    for (size_t s2 = 0; s2 < stage1.size() && finalists.size() < n_final; ++s2)
      if (!taken[s2]) finalists.push_back(stage1[s2].second);
  }
  // (banded candidates differ mostly in their lane patterns, which the
  // model ranks only to a few percent: time more of them)
  const size_t n_banded = (size_t)knob_long("ISD_TUNE_BANDED", 8);
  for (size_t b = 0; b < banded.size() && b < n_banded; ++b)
    finalists.push_back(banded[b]);
  // the finalists' NVRTC kernels compile concurrently (or come from the
  // cubin cache) before the first is timed
  if (jit_ok) {
    std::vector<HoistParams> ps;
    for (size_t i : finalists) {
      HoistParams hp;
      fill_hoist(lat, &cands[i], &hp);
      ps.push_back(hp);
    }
    jit_prefetch(ps);
  }
  float best_ms = 1e30f;
  bool steady = true;
  size_t best = finalists.empty() ? 0 : finalists[0];
  for (size_t i : finalists) {
    HoistParams hp;
    fill_hoist(lat, &cands[i], &hp);
    uint64_t run0, run1;
    run_range(cands[i].k, &run0, &run1);
    const uint64_t body = run1 - run0;
    uint64_t span_bits = hp.lane_mask;
    for (int v = 0; v < 5; ++v) span_bits |= hp.lane_vec[v];
    const uint64_t blk = 1ull << lane_span(span_bits);
    uint64_t len = (kTuneSliceConfigs >> hp.k);
    if (len > body) len = body;
    uint64_t off;
    if (hp.band_rows) {  // an aligned power-of-two slice: whole items
      while (len & (len - 1)) len &= len - 1;
      off = 0;
    } else {
      len = (len / blk) * blk;
      off = ((body - len) / 2 / blk) * blk;
    }
    if (len == 0) continue;
    hp.run_begin = run0 + off;
    hp.run_end = hp.run_begin + len;
    hp.hi_step = 1;
    // (banded candidates are timed with the cost-weighted item cut the walk
    // will use: equal-size items add a plan-dependent imbalance of a few
    // percent, enough to rank two lane patterns the wrong way round)
    if (set_band_launch(lat, cands[i], &hp, sms, true)) continue;
    if (hp.band_claim &&
        cudaMemsetAsync(reinterpret_cast<void*>(hp.band_claim), 0,
                        sizeof(uint32_t), st) != cudaSuccess)
      continue;
    float ms = 0.f;
    // (warm the finalist's kernel first: the JIT compile is not timed)
    int x = 0;
    if (jit_ok) {
      std::string why;
      HoistParams warm = hp;
      if (!warm.band_rows) warm.run_end = warm.run_begin + blk;
      x = launch_hoisted_jit(warm, scratch, sms, st, &why);
      if (x > 0) bump_launches(1);
    }
    // best of two timed launches: one noisy timing picked a plan ~9%
    // slower on c4 once (31.1 vs 33.9e12 configs/s)
    ms = 1e30f;
    float slowest = 0.f;
    for (int rep = 0; rep < 2; ++rep) {
      float t = 0.f;
      cudaEventRecord(e0, st);
      if (x > 0)
        launch_hoisted_jit(hp, scratch, sms, st, nullptr);
      else
        launch_hoisted(hp, scratch, sms, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&t, e0, e1);
      bump_launches(1);
      ms = std::min(ms, t);
      slowest = std::max(slowest, t);
    }
    const bool unsteady = slowest > 1.15f * ms;
    ms /= (float)len * (float)(1ull << hp.k);  // per configuration
    if (ms < best_ms) {
      best_ms = ms;
      best = i;
      steady = !unsteady;
    }
  }
  // the winner's work items, balanced by measurement over its own range
  if (!finalists.empty() && cands[best].band_rows) {
    HoistParams hp;
    fill_hoist(lat, &cands[best], &hp);
    uint64_t run0, run1;
    run_range(cands[best].k, &run0, &run1);
    uint64_t len = std::min<uint64_t>(kTuneSliceConfigs >> hp.k, run1 - run0);
    while (len & (len - 1)) len &= len - 1;
    if (len) {
      hp.run_begin = run0;
      hp.run_end = run0 + len;
      hp.hi_step = 1;
      calibrate_items(lat, cands[best], hp, sms, scratch, st, jit_ok);
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(scratch);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  cudaGetLastError();
  std::lock_guard<std::mutex> lock(g_plan_mu);
  PlanEntry& pe = g_plans[key];
  pe.info = cands[best];
  *info = pe.info;
  return steady;
}

// The best plan the model found without a banded table (banded plans need
// an aligned power-of-two range).
static bool unbanded_plan(const isd_lattice* lat, uint64_t hint,
                          isd_plan_info* info, uint64_t top) {
  std::lock_guard<std::mutex> lock(g_plan_mu);
  auto it = g_plans.find(plan_key(lat, hint, top));
  if (it == g_plans.end()) return false;
  const isd_plan_info* best = nullptr;
  for (const isd_plan_info& x : it->second.ranked)
    if (!x.band_rows && (!best || x.est_per_config < best->est_per_config))
      best = &x;
  if (!best) return false;
  *info = *best;
  return true;
}

// Identity of the current device for the plan cache: its name, SM count
// (as the grids are sized) and compute capability.
static std::string device_identity(int sms) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static std::map<int, std::string> names;
  std::string name;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = names.find(dev);
    if (it == names.end()) {
      cudaDeviceProp prop;
      std::string n = "?";
      if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess)
        n = std::string(prop.name) + "|cc" + std::to_string(prop.major) +
            std::to_string(prop.minor) + "|sm" +
            std::to_string(prop.multiProcessorCount);
      cudaGetLastError();
      it = names.emplace(dev, n).first;
    }
    name = it->second;
  }
  return name + "|grid" + std::to_string(sms);
}

// The plan of a walk over [start, end) (aligned power-of-two ranges hold
// their top bits fixed: `top` is their start).  Small walks take the host
// model's plan.  Walks of >= 2^33 configurations take the autotuned plan:
// from this process's memory, else from the disk cache (cache.cpp), else
// the model's candidates are timed now and the winner is written to the
// cache.  Tuning is skipped (the model's plan is used, not remembered as
// tuned) when `capturing`: a stream being captured into a graph cannot run
// the synchronous timing launches.  Returns 0, or > 0 when the lattice is
// too small for the hoisted kernel, or < 0 on error.
static int walk_plan(const isd_lattice* lat, uint64_t start, uint64_t end,
                     int sms, bool capturing, isd_plan_info* info,
                     uint64_t* top_out) {
  const uint64_t len = end - start;
  const uint64_t top = (!(len & (len - 1)) && start % len == 0 &&
                        knob_long("ISD_PLAN_TOP", 1) != 0)
                           ? start
                           : 0;
  *top_out = top;
  const bool large = len >= kTuneConfigs;
  const std::string key = plan_key(lat, len, top);
  {
    std::lock_guard<std::mutex> lock(g_plan_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end() && (it->second.tuned || it->second.rc || !large)) {
      *info = it->second.info;
      return it->second.rc;
    }
  }
  const bool tune = large && knob_long("ISD_AUTOTUNE", 1) != 0;
  const std::string dkey = key + "|" + device_identity(sms) + "|span" +
                           std::to_string(end - start);
  if (tune) {
    std::string blob;
    if (cache_get("plan", dkey, &blob) && blob.size() >= 4) {
      uint32_t n = 0;
      std::memcpy(&n, blob.data(), 4);
      if (n >= 1 && n <= 2 && blob.size() == 4 + n * sizeof(isd_plan_info)) {
        PlanEntry pe;
        std::memcpy(&pe.info, blob.data() + 4, sizeof(isd_plan_info));
        for (uint32_t i = 1; i < n; ++i) {
          isd_plan_info x;
          std::memcpy(&x, blob.data() + 4 + i * sizeof(isd_plan_info),
                      sizeof x);
          pe.ranked.push_back(x);
        }
        pe.tuned = true;
        std::lock_guard<std::mutex> lock(g_plan_mu);
        auto it = g_plans.find(key);
        if (it == g_plans.end() || !it->second.tuned)
          g_plans[key] = std::move(pe);
        *info = g_plans[key].info;
        return 0;
      }
    }
  }
  const int rc = cached_plan(lat, len, info, top);
  if (rc || !tune || capturing) return rc;
  if (!autotune(lat, len, start, end, sms, info, top)) return 0;
  // remember the winner (and the best unbanded plan, for unaligned ranges)
  std::string blob(4, '\0');
  uint32_t n = 1;
  blob.append(reinterpret_cast<const char*>(info), sizeof *info);
  isd_plan_info ub;
  {
    std::lock_guard<std::mutex> lock(g_plan_mu);
    const isd_plan_info* best = nullptr;
    for (const isd_plan_info& x : g_plans[key].ranked)
      if (!x.band_rows && (!best || x.est_per_config < best->est_per_config))
        best = &x;
    if (best) {
      ub = *best;
      ++n;
    }
  }
  if (n == 2) blob.append(reinterpret_cast<const char*>(&ub), sizeof ub);
  std::memcpy(&blob[0], &n, 4);
  cache_put("plan", dkey, blob);
  return 0;
}

// ---- walks as lists of stream operations ----------------------------------
// A walk is prepared first — validation, plan (and a first large walk's
// autotune), band work items, NVRTC kernels, all host-side and synchronous —
// into a list of operations, which are then issued back to back on a stream.
// So a caller's timing events around the issue see only device work, and
// several devices' walks can be prepared before any of them starts.
struct Op {
  const char* what;
  std::function<int(cudaStream_t)> fn;  // launches (>= 0) or -cudaError_t
};

static int issue_ops(const std::vector<Op>& ops, cudaStream_t st,
                     int* launches) {
  int nl = 0;
  for (const Op& op : ops) {
    const int r = op.fn(st);
    if (r < 0) return cuda_fail((cudaError_t)(-r), op.what);
    nl += r;
  }
  if (launches) *launches = nl;
  return ISD_OK;
}

static void prepare_canonical(const isd_lattice* lat, uint64_t a, uint64_t b,
                              unsigned long long* out, int sms,
                              bool small_grid, std::vector<Op>* ops) {
  CanonParams p;
  fill_canon(lat, &p);
  const uint64_t cap = launch_cap(sms);
  while (a < b) {
    const uint64_t e = (b - a > cap) ? a + cap : b;
    p.start = a;
    p.end = e;
    ops->push_back({"k1_canonical launch", [p, out, sms, small_grid](
                                               cudaStream_t st) {
                      return launch_canonical(p, out, sms, st, small_grid);
                    }});
    a = e;
  }
}

static int prepare_walk(const isd_lattice* lat, uint64_t start, uint64_t end,
                        int algo, unsigned long long* out, int accumulate,
                        bool capturing, std::vector<Op>* ops);

// Half walk + mirror (ISD_FLAG_FLIP_SYMMETRY).
static int prepare_flip(const isd_lattice* lat, uint64_t start, uint64_t end,
                        int algo, unsigned long long* out, int accumulate,
                        bool capturing, std::vector<Op>* ops) {
  const uint64_t total = 1ull << lat->n_spins;
  if (start != 0 || end != total)
    return fail(ISD_EINVAL, "flip symmetry needs the full range [0, 2^N)");
  if (accumulate)
    return fail(ISD_EINVAL, "flip symmetry cannot accumulate into a table");
  int rc = prepare_walk(lat, 0, total / 2, algo & 0xff, out, 0, capturing, ops);
  if (rc) return rc;
  const uint32_t n = lat->n_spins, b = lat->n_bonds;
  ops->push_back({"k3_mirror launch", [out, n, b](cudaStream_t st) {
                    return launch_mirror(out, n, b, st);
                  }});
  return ISD_OK;
}

static int prepare_walk(const isd_lattice* lat, uint64_t start, uint64_t end,
                        int algo, unsigned long long* out, int accumulate,
                        bool capturing, std::vector<Op>* ops) {
  NvtxRange nvtx("isd:prepare walk");
  char err[256];
  int rc = validate_lattice(lat, err, sizeof err);
  if (rc) return fail(rc, "%s", err);
  if (algo & ISD_FLAG_FLIP_SYMMETRY)
    return prepare_flip(lat, start, end, algo, out, accumulate, capturing,
                        ops);
  const uint64_t total = 1ull << lat->n_spins;
  if (!(start <= end && end <= total))
    return fail(ISD_EINVAL, "range [%llu, %llu) invalid for 2^%u configurations",
                (unsigned long long)start, (unsigned long long)end,
                lat->n_spins);
  if (algo < ISD_ALGO_AUTO || algo > ISD_ALGO_HOISTED)
    return fail(ISD_EINVAL, "unknown algo %d", algo);
  if (!out) return fail(ISD_EINVAL, "counts pointer is NULL");
  const size_t bytes =
      (size_t)(lat->n_spins + 1) * (lat->n_bonds + 1) * sizeof(uint64_t);
  if (!accumulate)
    ops->push_back({"cudaMemsetAsync", [out, bytes](cudaStream_t st) {
                      const cudaError_t e = cudaMemsetAsync(out, 0, bytes, st);
                      return e == cudaSuccess ? 0 : -(int)e;
                    }});
  if (start == end) return ISD_OK;
  int sms = 0;
  rc = current_sm_count(&sms);
  if (rc) return rc;

  if (algo == ISD_ALGO_CANONICAL) {
    g_kernel_info = "k1_canonical";
    prepare_canonical(lat, start, end, out, sms, false, ops);
    return ISD_OK;
  }
  isd_plan_info info;
  // an aligned power-of-two range (a shard) holds its top bits fixed:
  // the layout model sees them (ISD_PLAN_TOP=0: plan as for shard 0)
  uint64_t top = 0;
  const int too_small =
      walk_plan(lat, start, end, sms, capturing, &info, &top);
  if (too_small < 0) return too_small;
  if (too_small) {
    if (algo == ISD_ALGO_HOISTED)
      return fail(ISD_EINVAL, "lattice of %u spins too small for the hoisted "
                  "kernel", lat->n_spins);
    g_kernel_info = "k1_canonical";
    prepare_canonical(lat, start, end, out, sms, true, ops);
    return ISD_OK;
  }
  // a banded plan runs only on an aligned power-of-two range
  if (info.band_rows && !band_ok(info, start, end) &&
      !unbanded_plan(lat, end - start, &info, top))
    return fail(ISD_EINVAL, "no unbanded plan for an unaligned range");
  const uint32_t k = info.k;
  const uint64_t r0 = (start + ((1ull << k) - 1)) >> k;
  const uint64_t r1 = end >> k;
  if (r0 >= r1) {
    g_kernel_info = "k1_canonical";
    prepare_canonical(lat, start, end, out, sms, true, ops);
    return ISD_OK;
  }
  // unaligned head and tail: fewer than 2^k configurations each
  if (start < (r0 << k))
    prepare_canonical(lat, start, r0 << k, out, sms, true, ops);
  // experiment knob: ISD_LAYOUT="A,B,P,ls[,lanemask_hex]" forces the
  // histogram layout and lane placement (window at ls, or the mask)
  std::string lay_s;
  if (knob_str("ISD_LAYOUT", &lay_s) && !lay_s.empty()) {
    const char* lay = lay_s.c_str();
    unsigned a = 0, b = 0, pw = 0, ls = 0;
    unsigned long long mask = 0;
    const int got = std::sscanf(lay, "%u,%u,%u,%u,%llx", &a, &b, &pw, &ls, &mask);
    if (got >= 4 && a && b) {
      info.row_words = a;
      info.e_words = b;
      info.plane_words = pw;
      info.lane_mask = (got == 5 && mask) ? mask : (0x1Full << ls);
      uint64_t m = info.lane_mask;
      for (int v = 0; v < 5; ++v) {
        info.lane_vec[v] = m & (~m + 1);
        m ^= info.lane_vec[v];
      }
      info.hist_words = lat->n_spins * a + lat->n_bonds * b + pw + 1;
      info.base_words = info.hist_words;
      info.pair_mode = 0;  // the knob describes an unpaired layout
      info.band_rows = 0;
    }
  }
  HoistParams hp;
  fill_hoist(lat, &info, &hp);
  // A small walk is bound by what every block does once — zero its tables,
  // flush them — not by the walk: one table per block instead of up to 16
  // privatised copies (c2, 2^25 configurations: 30 -> 22 us; c1 25 -> 15)
  if (end - start <= (1ull << 26))
    hp.n_hist = 1;
  else if (end - start <= (1ull << 28) && hp.n_hist > 2)
    hp.n_hist = 2;
  const uint64_t runs_per_launch = launch_cap(sms) >> k;
  // large walks use the per-lattice NVRTC specialisation (jit.cpp)
  // (ISD_JIT=0: never; ISD_JIT=2: for every hoisted walk — tests)
  const long jit_mode = knob_long("ISD_JIT", 1);
  bool use_jit = jit_mode != 0 && (end - start >= kTuneConfigs || jit_mode == 2);
  if (use_jit) {
    std::string why;
    if (!jit_ready(hp, &why)) {  // NVRTC unavailable: same arithmetic, AOT
      use_jit = false;
      g_kernel_info = "k1_hoisted_aot (jit unavailable: " + why + ")";
    } else {
      g_kernel_info = "k1_hoisted_jit";
    }
  } else {
    g_kernel_info = "k1_hoisted_aot";
  }
  for (uint64_t r = r0; r < r1;) {
    const uint64_t re = (r1 - r > runs_per_launch) ? r + runs_per_launch : r1;
    hp.run_begin = r;
    hp.run_end = re;
    // the plan's lane placement tiles the launch only if its run count is a
    // multiple of 2^lane_span; otherwise lanes take the lowest 5 run bits
    hp.lane_mask = info.lane_mask;
    for (int v = 0; v < 5; ++v) hp.lane_vec[v] = info.lane_vec[v];
    uint64_t span_bits = hp.lane_mask;
    for (int v = 0; v < 5; ++v) span_bits |= hp.lane_vec[v];
    if ((re - r) & ((1ull << lane_span(span_bits)) - 1))
      default_lanes(&hp.lane_mask, hp.lane_vec);
    hp.hi_step = 1;
    rc = set_band_launch(lat, info, &hp, sms);
    if (rc) return rc;
    if (hp.band_claim) {  // (dynamic item claims: zero the counter first)
      void* claim = reinterpret_cast<void*>(hp.band_claim);
      ops->push_back({"band claim counter reset", [claim](cudaStream_t st) {
                        const cudaError_t e =
                            cudaMemsetAsync(claim, 0, sizeof(uint32_t), st);
                        return e == cudaSuccess ? 0 : -(int)e;
                      }});
    }
    if (use_jit)
      ops->push_back({"k1_jit launch", [hp, out, sms](cudaStream_t st) {
                        const int x =
                            launch_hoisted_jit(hp, out, sms, st, nullptr);
                        // (0: the kernel vanished after jit_ready said yes)
                        return x == 0 ? -(int)cudaErrorInvalidDeviceFunction
                                      : x;
                      }});
    else
      ops->push_back({"k1_hoisted launch", [hp, out, sms](cudaStream_t st) {
                        return launch_hoisted(hp, out, sms, st);
                      }});
    r = re;
  }
  if ((r1 << k) < end)
    prepare_canonical(lat, r1 << k, end, out, sms, true, ops);
  return ISD_OK;
}

// Prepared walks are memoised: a repeated walk (same lattice, range, algo,
// table and device, same knobs) reuses its operation list instead of
// rebuilding plan keys, band items and kernel lookups on every call (tens
// of microseconds of host time on the e2e path).  Only fully tuned walks are
// kept; knob changes and installed plans clear the memo.
struct PreparedWalk {
  std::vector<Op> ops;
  std::string kernel_info;
};
static std::mutex g_prep_mu;
static std::map<std::string, PreparedWalk> g_prep;

static void forget_prepared() {
  std::lock_guard<std::mutex> lock(g_prep_mu);
  g_prep.clear();
}

static int prepare_walk_cached(const isd_lattice* lat, uint64_t start,
                               uint64_t end, int algo,
                               unsigned long long* out, int accumulate,
                               bool capturing, std::vector<Op>* ops) {
  int dev = -1;
  cudaGetDevice(&dev);
  std::string key(reinterpret_cast<const char*>(lat), sizeof(*lat));
  char buf[160];
  std::snprintf(buf, sizeof buf, "|%llu|%llu|%d|%d|%p|%d",
                (unsigned long long)start, (unsigned long long)end, algo,
                accumulate, (void*)out, dev);
  key += buf;
  key += knob_signature();
  if (!capturing) {
    std::lock_guard<std::mutex> lock(g_prep_mu);
    auto it = g_prep.find(key);
    if (it != g_prep.end()) {
      ops->insert(ops->end(), it->second.ops.begin(), it->second.ops.end());
      g_kernel_info = it->second.kernel_info;
      return ISD_OK;
    }
  }
  std::vector<Op> mine;
  const int rc =
      prepare_walk(lat, start, end, algo, out, accumulate, capturing, &mine);
  if (rc) return rc;
  // keep it only when the plan is final: a large walk's plan must be tuned
  // (not the model's stand-in used while capturing), and no op may depend
  // on per-launch state (dynamic item claims reset a counter slot)
  bool keep = !capturing;
  for (const Op& op : mine)
    keep = keep && std::strcmp(op.what, "band claim counter reset") != 0;
  if (keep) {
    std::lock_guard<std::mutex> lock(g_prep_mu);
    if (g_prep.size() >= 256) g_prep.clear();
    g_prep[key] = PreparedWalk{mine, g_kernel_info};
  }
  ops->insert(ops->end(), mine.begin(), mine.end());
  return ISD_OK;
}

static bool stream_capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cap != cudaStreamCaptureStatusNone;
}

static int enumerate_impl(const isd_lattice* lat, uint64_t start,
                          uint64_t end, int algo, unsigned long long* out,
                          int accumulate, cudaStream_t st, int* launches) {
  std::vector<Op> ops;
  const int rc = prepare_walk_cached(lat, start, end, algo, out, accumulate,
                                     stream_capturing(st), &ops);
  if (rc) return rc;
  return issue_ops(ops, st, launches);
}

// ---- multi-device walks ----------------------------------------------------
// One process drives several GPUs (enumeration.py:365-390's Pool and root sum,
// PAPER.md:98-115's MPI reduce): each device walks its shards into its own
// table on its own stream; the root device then reads every table over
// NVLink (peer access) inside one kernel that forms the combined table — K4,
// or K2a when thermodynamics follow (launch_thermo_set) — so no host sum and
// no separate reduce launch.  Where peer access is unavailable the root
// copies that table first (cudaMemcpyPeerAsync, still device to device).

// Peer access from `root` to `dev` (enabled once per pair): true when the
// root's kernels may read dev's memory directly.
static bool peer_access(int root, int dev) {
  if (root == dev) return true;
  static std::mutex mu;
  static std::map<std::pair<int, int>, bool> known;
  std::lock_guard<std::mutex> lock(mu);
  auto it = known.find({root, dev});
  if (it != known.end()) return it->second;
  int can = 0;
  bool ok = false;
  if (cudaDeviceCanAccessPeer(&can, root, dev) == cudaSuccess && can) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(root);
    const cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
    ok = e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled;
    cudaGetLastError();
    cudaSetDevice(cur);
  }
  cudaGetLastError();
  known[{root, dev}] = ok;
  return ok;
}

// The reference's partition of [start, end) into n contiguous shards
// (make_shards, enumeration.py:44-63: the first (end - start) mod n shards
// are one longer; for n = 2^k over an aligned power-of-two range they are
// the top-k-bit prefixes).
static void split_range(uint64_t start, uint64_t end, int n,
                        std::vector<uint64_t>* edge) {
  const uint64_t len = end - start, q = len / (uint64_t)n,
                 r = len % (uint64_t)n;
  edge->resize(n + 1);
  for (int i = 0; i <= n; ++i)
    (*edge)[i] = start + (uint64_t)i * q + std::min<uint64_t>((uint64_t)i, r);
}

// The thermodynamic grid a multi-device walk evaluates on the root right
// after the combine (isd_enumerate_thermo): host inputs and output.
struct ThermoReq {
  double scale;
  const double* fields;
  int n_fields;
  const double* temps;
  int n_temps;
  double* out_host;
};

static int enumerate_multi(const isd_lattice* lat, uint64_t start,
                           uint64_t end, int n_shards, const int* devs,
                           int algo, uint64_t* counts_host, double* shard_ms,
                           double* total_ms, const ThermoReq* thermo = nullptr) {
  NvtxRange nvtx("isd:enumerate_multi");
  char err[256];
  int rc = validate_lattice(lat, err, sizeof err);
  if (rc) return fail(rc, "%s", err);
  if (n_shards < 1 || !devs)
    return fail(ISD_EINVAL, "need n_shards >= 1 and a device list");
  if (!counts_host) return fail(ISD_EINVAL, "counts pointer is NULL");
  const uint64_t total = 1ull << lat->n_spins;
  if (!(start <= end && end <= total))
    return fail(ISD_EINVAL, "range [%llu, %llu) invalid for 2^%u configurations",
                (unsigned long long)start, (unsigned long long)end,
                lat->n_spins);
  const bool flip = (algo & ISD_FLAG_FLIP_SYMMETRY) != 0;
  uint64_t wstart = start, wend = end;
  if (flip) {  // shards of the top-spin-down half, mirrored on the root
    if (start != 0 || end != total)
      return fail(ISD_EINVAL, "flip symmetry needs the full range [0, 2^N)");
    wend = total / 2;
  }
  if ((uint64_t)n_shards > std::max<uint64_t>(wend - wstart, 1))
    return fail(ISD_EINVAL, "%d shards for %llu configurations", n_shards,
                (unsigned long long)(wend - wstart));
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(ISD_ENODEV, "no CUDA device available (%s)",
                e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  std::vector<int> uniq;  // distinct devices, root (devs[0]) first
  for (int i = 0; i < n_shards; ++i) {
    if (devs[i] < 0 || devs[i] >= ndev || devs[i] >= 64)
      return fail(ISD_ENODEV, "device %d outside [0, %d)", devs[i], ndev);
    if (std::find(uniq.begin(), uniq.end(), devs[i]) == uniq.end())
      uniq.push_back(devs[i]);
  }
  if ((int)uniq.size() > kMaxTables)
    return fail(ISD_EINVAL, "more than %d distinct devices", kMaxTables);
  const int root = devs[0];
  DeviceGuard guard;
  // lock every device involved, in ascending order (no lock-order cycles
  // with concurrent multi-device calls)
  std::vector<int> order(uniq);
  std::sort(order.begin(), order.end());
  std::vector<std::unique_lock<std::mutex>> locks(order.size());
  for (size_t j = 0; j < order.size(); ++j) {
    DevState* s = nullptr;
    rc = get_dev(order[j], &s, &locks[j]);
    if (rc) return rc;
  }
  const size_t bytes =
      (size_t)(lat->n_spins + 1) * (lat->n_bonds + 1) * sizeof(uint64_t);
  for (int d : uniq) {
    cudaSetDevice(d);
    DevState& s = g_dev[d];
    rc = ensure_buffer(&s.d_counts, &s.d_counts_bytes, bytes,
                       "cudaMalloc(counts)");
    if (rc) return rc;
  }
  cudaSetDevice(root);
  DevState& R = g_dev[root];
  rc = ensure_buffer(&R.d_sum, &R.d_sum_bytes, bytes, "cudaMalloc(sum)");
  if (rc) return rc;
  rc = ensure_buffer(&R.d_copies, &R.d_copies_bytes, bytes * uniq.size(),
                     "cudaMalloc(table copies)");
  if (rc) return rc;
  // the grid, if any: [fields | temps | results] in the root's d_buf, the
  // inputs copied up at the start (they overlap the walks)
  const size_t n_pts = thermo ? (size_t)thermo->n_fields * thermo->n_temps : 0;
  const size_t grid_in = thermo ? (size_t)(thermo->n_fields + thermo->n_temps) * 8 : 0;
  const size_t grid_out = n_pts * ISD_THERMO_FIELDS * 8;
  if (n_pts) {
    rc = ensure_buffer(&R.d_buf, &R.d_buf_bytes, grid_in + grid_out,
                       "cudaMalloc(thermo)");
    if (rc) return rc;
  }
  std::vector<uint64_t> edge;
  split_range(wstart, wend, n_shards, &edge);

  // 1. prepare every shard's walk, one host thread per device (plans, a
  // first large walk's autotune and NVRTC compiles run concurrently)
  std::vector<std::vector<Op>> ops(n_shards);
  std::vector<int> prc(uniq.size(), 0);
  std::vector<std::string> perr(uniq.size()), kinfo(uniq.size());
  auto prepare_dev = [&](size_t j) {
    const int d = uniq[j];
    cudaSetDevice(d);
    bool first = true;
    for (int i = 0; i < n_shards && !prc[j]; ++i) {
      if (devs[i] != d) continue;
      prc[j] = prepare_walk_cached(lat, edge[i], edge[i + 1], algo & 0xff,
                                   g_dev[d].d_counts, first ? 0 : 1, false,
                                   &ops[i]);
      first = false;
      if (prc[j]) perr[j] = g_err;
    }
    kinfo[j] = g_kernel_info;
  };
  if (uniq.size() == 1) {
    prepare_dev(0);
  } else {
    std::vector<std::thread> pool;
    for (size_t j = 0; j < uniq.size(); ++j) pool.emplace_back(prepare_dev, j);
    for (std::thread& t : pool) t.join();
  }
  for (size_t j = 0; j < uniq.size(); ++j)
    if (prc[j]) return fail(prc[j], "%s", perr[j].c_str());
  g_kernel_info = kinfo[0];

  // 2. issue: every device starts after the root's start event; each
  // shard is bracketed by its own events on its device's stream
  std::vector<cudaEvent_t> es(n_shards), ee(n_shards), done(uniq.size());
  auto destroy_events = [&]() {
    for (int i = 0; i < n_shards; ++i) {
      if (es[i]) cudaEventDestroy(es[i]);
      if (ee[i]) cudaEventDestroy(ee[i]);
    }
    for (cudaEvent_t x : done)
      if (x) cudaEventDestroy(x);
  };
  std::fill(es.begin(), es.end(), nullptr);
  std::fill(ee.begin(), ee.end(), nullptr);
  std::fill(done.begin(), done.end(), nullptr);
  cudaSetDevice(root);
  void* stage = nullptr;
  rc = stage_buffer(&R, bytes + grid_in + grid_out, &stage);
  if (rc) return rc;
  char* hs = static_cast<char*>(stage);
  cudaEventRecord(R.ev0, R.stream);
  if (n_pts) {
    std::memcpy(hs + bytes, thermo->fields, (size_t)thermo->n_fields * 8);
    std::memcpy(hs + bytes + (size_t)thermo->n_fields * 8, thermo->temps,
                (size_t)thermo->n_temps * 8);
    e = cudaMemcpyAsync(R.d_buf, hs + bytes, grid_in, cudaMemcpyHostToDevice,
                        R.stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(grid)");
  }
  int nl = 0;
  for (size_t j = 0; j < uniq.size(); ++j) {
    const int d = uniq[j];
    cudaSetDevice(d);
    cudaStream_t st = g_dev[d].stream;
    if (d != root) cudaStreamWaitEvent(st, R.ev0, 0);
    for (int i = 0; i < n_shards; ++i) {
      if (devs[i] != d) continue;
      cudaEventCreate(&es[i]);
      cudaEventCreate(&ee[i]);
      cudaEventRecord(es[i], st);
      int x = 0;
      rc = issue_ops(ops[i], st, &x);
      nl += x;
      if (rc) {
        destroy_events();
        return rc;
      }
      cudaEventRecord(ee[i], st);
    }
    cudaEventCreateWithFlags(&done[j], cudaEventDisableTiming);
    cudaEventRecord(done[j], st);
  }
  // 3. combine on the root: one kernel reads every device's table (none
  // when the root walked everything itself: its table is the result)
  cudaSetDevice(root);
  TableSet tabs;
  tabs.n = (int)uniq.size();
  unsigned long long* result = R.d_sum;
  for (size_t j = 0; j < uniq.size(); ++j) {
    const int d = uniq[j];
    if (d != root) cudaStreamWaitEvent(R.stream, done[j], 0);
    // (ISD_PEER=0: take the copy path even where the root could read the
    // table directly — how the one-GPU pool tests it)
    if (knob_long("ISD_PEER", 1) != 0 && peer_access(root, d)) {
      tabs.t[j] = g_dev[d].d_counts;
    } else {
      unsigned long long* copy = R.d_copies + j * (bytes / 8);
      e = cudaMemcpyPeerAsync(copy, root, g_dev[d].d_counts, d, bytes,
                              R.stream);
      if (e != cudaSuccess) {
        destroy_events();
        return cuda_fail(e, "cudaMemcpyPeerAsync");
      }
      tabs.t[j] = copy;
    }
  }
  int r = 0;
  if (tabs.n == 1 && tabs.t[0] == g_dev[root].d_counts)
    result = g_dev[root].d_counts;
  else
    r = launch_gather(tabs, R.d_sum, lat->n_spins, lat->n_bonds, R.stream);
  if (r >= 0 && flip) {
    const int r2 = launch_mirror(result, lat->n_spins, lat->n_bonds, R.stream);
    r = r2 < 0 ? r2 : r + r2;
  }
  if (r >= 0 && n_pts) {
    const double* d_f = reinterpret_cast<const double*>(R.d_buf);
    const double* d_t = d_f + thermo->n_fields;
    double* d_o = R.d_buf + thermo->n_fields + thermo->n_temps;
    const int r3 = launch_thermo(result, lat->n_spins, lat->n_bonds,
                                 thermo->scale, d_f, thermo->n_fields, d_t,
                                 thermo->n_temps, d_o, R.stream);
    r = r3 < 0 ? r3 : r + r3;
  }
  if (r < 0) {
    destroy_events();
    return cuda_fail((cudaError_t)(-r), "k4 / k2 launch");
  }
  nl += r;
  bump_launches((uint64_t)nl);
  cudaEventRecord(R.ev1, R.stream);
  e = cudaMemcpyAsync(stage, result, bytes, cudaMemcpyDeviceToHost, R.stream);
  if (e == cudaSuccess && n_pts)
    e = cudaMemcpyAsync(hs + bytes + grid_in,
                        R.d_buf + thermo->n_fields + thermo->n_temps, grid_out,
                        cudaMemcpyDeviceToHost, R.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(R.stream);
  if (e != cudaSuccess) {
    destroy_events();
    return cuda_fail(e, "multi-device enumeration");
  }
  std::memcpy(counts_host, stage, bytes);
  if (n_pts) std::memcpy(thermo->out_host, hs + bytes + grid_in, grid_out);
  for (int i = 0; i < n_shards; ++i) {
    float ms = 0.f;
    cudaSetDevice(devs[i]);
    cudaEventElapsedTime(&ms, es[i], ee[i]);
    if (shard_ms) shard_ms[i] = ms;
  }
  cudaSetDevice(root);
  if (total_ms) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, R.ev0, R.ev1);
    *total_ms = ms;
  }
  destroy_events();
  return ISD_OK;
}

}  // namespace isd

using namespace isd;

extern "C" {

int isd_validate(const isd_lattice* lat) {
  char err[256];
  int rc = validate_lattice(lat, err, sizeof err);
  if (rc) return fail(rc, "%s", err);
  return ISD_OK;
}

int isd_plan(const isd_lattice* lat, uint64_t n_configs_hint,
             isd_plan_info* out) {
  int rc = isd_validate(lat);
  if (rc) return rc;
  if (!out) return fail(ISD_EINVAL, "plan pointer is NULL");
  return cached_plan(lat, n_configs_hint, out);
}

int isd_walk_plan(const isd_lattice* lat, uint64_t start, uint64_t end,
                  int device, isd_plan_info* out) {
  int rc = isd_validate(lat);
  if (rc) return rc;
  if (!out) return fail(ISD_EINVAL, "plan pointer is NULL");
  if (!(start < end && end <= (1ull << lat->n_spins)))
    return fail(ISD_EINVAL, "range [%llu, %llu) invalid for 2^%u configurations",
                (unsigned long long)start, (unsigned long long)end,
                lat->n_spins);
  DeviceGuard guard;
  DevState* s = nullptr;
  std::unique_lock<std::mutex> lock;
  rc = get_dev(device, &s, &lock);
  if (rc) return rc;
  int sms = 0;
  rc = current_sm_count(&sms);
  if (rc) return rc;
  uint64_t top = 0;
  rc = walk_plan(lat, start, end, sms, false, out, &top);
  if (rc) return rc;
  if (out->band_rows && !band_ok(*out, start, end) &&
      !unbanded_plan(lat, end - start, out, top))
    return fail(ISD_EINVAL, "no unbanded plan for an unaligned range");
  return ISD_OK;
}

int isd_set_walk_plan(const isd_lattice* lat, uint64_t start, uint64_t end,
                      const isd_plan_info* plan) {
  int rc = isd_validate(lat);
  if (rc) return rc;
  if (!plan) return fail(ISD_EINVAL, "plan pointer is NULL");
  if (!(start < end && end <= (1ull << lat->n_spins)))
    return fail(ISD_EINVAL, "range [%llu, %llu) invalid for 2^%u configurations",
                (unsigned long long)start, (unsigned long long)end,
                lat->n_spins);
  if (plan->u != ISD_COPY_BITS || plan->k != plan->u + plan->l ||
      plan->k > lat->n_spins || plan->pair_mode > 3 ||
      (size_t)plan->hist_words * 4 > 227 * 1024)
    return fail(ISD_EINVAL, "not a hoisted-kernel plan of this lattice");
  const uint64_t len = end - start;
  const uint64_t top = (!(len & (len - 1)) && start % len == 0 &&
                        knob_long("ISD_PLAN_TOP", 1) != 0)
                           ? start
                           : 0;
  isd_plan_info model;
  rc = cached_plan(lat, len, &model, top);  // (ranked list for fallbacks)
  if (rc) return fail(ISD_EINVAL, "lattice too small for the hoisted kernel");
  std::lock_guard<std::mutex> lock(g_plan_mu);
  PlanEntry& pe = g_plans[plan_key(lat, len, top)];
  pe.info = *plan;
  pe.tuned = true;
  forget_prepared();
  return ISD_OK;
}

int isd_band_costs(const isd_lattice* lat, const isd_plan_info* plan,
                   uint64_t run_begin, uint32_t run_bits, uint32_t n_seg,
                   uint32_t samples, double* out) {
  int rc = isd_validate(lat);
  if (rc) return rc;
  if (!plan || !out || n_seg < 1 || samples < 1 || run_bits < 6 ||
      run_bits > 28)
    return fail(ISD_EINVAL, "bad band cost arguments");
  std::vector<double> c;
  band_slot_cost(lat, *plan, run_begin, plan->lane_mask, plan->lane_vec,
                 (int)run_bits, (int)n_seg, (int)samples, &c);
  std::memcpy(out, c.data(), c.size() * sizeof(double));
  return (int)c.size();
}

int isd_band_slot_order(const isd_lattice* lat, const isd_plan_info* plan,
                        uint64_t run_begin, uint32_t run_bits, int reorder,
                        uint8_t* pos_out) {
  int rc = isd_validate(lat);
  if (rc) return rc;
  if (!plan || !pos_out || run_bits < 6 || run_bits > 28)
    return fail(ISD_EINVAL, "bad band order arguments");
  uint8_t pos[24] = {0};
  band_slot_order(lat, *plan, run_begin, plan->lane_mask, plan->lane_vec,
                  (int)run_bits, reorder != 0, pos);
  const int F = (int)run_bits - 5;
  uint32_t m[16], r[16];
  if (band_slot_fields(pos, F, m, r) < 0)
    return fail(ISD_EINVAL, "slot map needs too many fields");
  std::memcpy(pos_out, pos, (size_t)F);
  return F;
}

int isd_plan_range(const isd_lattice* lat, uint64_t start, uint64_t end,
                   isd_plan_info* out) {
  int rc = isd_validate(lat);
  if (rc) return rc;
  if (!out) return fail(ISD_EINVAL, "plan pointer is NULL");
  if (!(start < end && end <= (1ull << lat->n_spins)))
    return fail(ISD_EINVAL, "range [%llu, %llu) invalid for 2^%u configurations",
                (unsigned long long)start, (unsigned long long)end,
                lat->n_spins);
  const uint64_t len = end - start;
  const uint64_t top = (!(len & (len - 1)) && start % len == 0 &&
                        knob_long("ISD_PLAN_TOP", 1) != 0)
                           ? start
                           : 0;
  return cached_plan(lat, len, out, top);
}

int isd_band_items(uint32_t free_bits, uint32_t n_target, uint32_t span,
                   const double* seg_cost, uint32_t n_seg, double flush_units,
                   uint64_t* out, uint32_t max_items, uint32_t* n_items,
                   int* exact) {
  if (free_bits < 1 || free_bits > 23 || n_target < 1 || span > 8 ||
      (n_seg && !seg_cost) || !out || !n_items || !exact)
    return fail(ISD_EINVAL, "bad band item arguments");
  std::vector<double> w;
  if (n_seg) w.assign(seg_cost, seg_cost + n_seg);
  bool ex = false;
  const std::vector<BandItem> items = band_work_items(
      (int)free_bits, (int)n_target, (int)span, w, flush_units, &ex);
  if (items.size() > max_items) return fail(ISD_EINVAL, "out too small");
  for (size_t i = 0; i < items.size(); ++i) {
    out[3 * i] = items[i].g0;
    out[3 * i + 1] = items[i].g1;
    out[3 * i + 2] = items[i].q0;
  }
  *n_items = (uint32_t)items.size();
  *exact = ex ? 1 : 0;
  return ISD_OK;
}

int isd_jit_check(const isd_lattice* lat, uint64_t n_configs_hint,
                  uint64_t* cubin_bytes) {
  int rc = isd_validate(lat);
  if (rc) return rc;
  isd_plan_info info;
  if (cached_plan(lat, n_configs_hint, &info))
    return fail(ISD_EINVAL, "lattice too small for the hoisted kernel");
  HoistParams hp;
  fill_hoist(lat, &info, &hp);
  std::string why;
  const int n = jit_compile_check(hp, &why);
  if (n <= 0) return fail(ISD_ECUDA, "%s", why.c_str());
  if (cubin_bytes) *cubin_bytes = (uint64_t)n;
  return ISD_OK;
}

int isd_enumerate_async(const isd_lattice* lat, uint64_t start, uint64_t end,
                        int algo, uint64_t* counts_dev, int accumulate,
                        void* stream, int* launches) {
  int nl = 0;
  int rc = enumerate_impl(lat, start, end, algo,
                          reinterpret_cast<unsigned long long*>(counts_dev),
                          accumulate, (cudaStream_t)stream, &nl);
  bump_launches((uint64_t)nl);
  if (launches) *launches = nl;
  return rc;
}

int isd_enumerate(const isd_lattice* lat, uint64_t start, uint64_t end,
                  int device, int algo, uint64_t* counts_host,
                  double* device_ms) {
  NvtxRange nvtx("isd:enumerate");
  int rc = isd_validate(lat);
  if (rc) return rc;
  if (!counts_host) return fail(ISD_EINVAL, "counts pointer is NULL");
  DeviceGuard guard;
  DevState* s = nullptr;
  std::unique_lock<std::mutex> lock;
  rc = get_dev(device, &s, &lock);
  if (rc) return rc;
  const size_t bytes =
      (size_t)(lat->n_spins + 1) * (lat->n_bonds + 1) * sizeof(uint64_t);
  if (s->d_counts_bytes < bytes) {
    if (s->d_counts) cudaFree(s->d_counts);
    s->d_counts = nullptr;
    s->d_counts_bytes = 0;
    cudaError_t e = cudaMalloc(&s->d_counts, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(counts)");
    s->d_counts_bytes = bytes;
  }
  // host-side preparation (plan, a first large walk's autotune, work
  // items, NVRTC kernels) happens before the timed region
  std::vector<Op> ops;
  rc = prepare_walk_cached(lat, start, end, algo, s->d_counts, 0, false,
                           &ops);
  if (rc) return rc;
  cudaEventRecord(s->ev0, s->stream);
  int nl = 0;
  rc = issue_ops(ops, s->stream, &nl);
  bump_launches((uint64_t)nl);
  if (rc) return rc;
  cudaEventRecord(s->ev1, s->stream);
  void* stage = nullptr;
  rc = stage_buffer(s, bytes, &stage);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(stage, s->d_counts, bytes,
                                  cudaMemcpyDeviceToHost, s->stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(D2H)");
  e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return cuda_fail(e, "enumeration kernels");
  std::memcpy(counts_host, stage, bytes);
  if (device_ms) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s->ev0, s->ev1);
    *device_ms = ms;
  }
  return ISD_OK;
}

int isd_enumerate_multi(const isd_lattice* lat, uint64_t start, uint64_t end,
                        int n_shards, const int* devs, int algo,
                        uint64_t* counts_host, double* shard_ms,
                        double* total_ms) {
  return enumerate_multi(lat, start, end, n_shards, devs, algo, counts_host,
                         shard_ms, total_ms);
}

int isd_enumerate_thermo(const isd_lattice* lat, uint64_t start, uint64_t end,
                         int n_shards, const int* devs, int algo,
                         double energy_scale, const double* fields,
                         int n_fields, const double* temps, int n_temps,
                         uint64_t* counts_host, double* out_host,
                         double* shard_ms, double* total_ms) {
  if (n_fields < 0 || n_temps < 0)
    return fail(ISD_EINVAL, "negative grid size");
  if (!(energy_scale > 0)) return fail(ISD_EINVAL, "energy_scale must be > 0");
  if (n_fields * n_temps > 0 && (!fields || !temps || !out_host))
    return fail(ISD_EINVAL, "NULL buffer");
  for (int i = 0; i < n_temps; ++i)
    if (!(temps[i] > 0)) return fail(ISD_EINVAL, "temperatures must be > 0");
  ThermoReq req{energy_scale, fields, n_fields, temps, n_temps, out_host};
  return enumerate_multi(lat, start, end, n_shards, devs, algo, counts_host,
                         shard_ms, total_ms, &req);
}

int isd_thermo_gather_async(const uint64_t* const* tables_dev, int n_tables,
                            uint64_t* sum_dev, uint32_t n_spins,
                            uint32_t n_bonds, double energy_scale,
                            const double* fields_dev, int n_fields,
                            const double* temps_dev, int n_temps,
                            double* out_dev, void* stream) {
  if (n_spins < 1 || n_spins > ISD_MAX_SPINS || n_bonds > 3 * ISD_MAX_SPINS)
    return fail(ISD_EINVAL, "bad table shape N=%u B=%u", n_spins, n_bonds);
  if (n_tables < 1 || n_tables > kMaxTables || !tables_dev)
    return fail(ISD_EINVAL, "need 1..%d tables", kMaxTables);
  if (n_fields < 0 || n_temps < 0)
    return fail(ISD_EINVAL, "negative grid size");
  if (!(energy_scale > 0)) return fail(ISD_EINVAL, "energy_scale must be > 0");
  const bool grid = n_fields * n_temps > 0;
  if ((grid && (!fields_dev || !temps_dev || !out_dev)) || (!grid && !sum_dev))
    return fail(ISD_EINVAL, "NULL buffer");
  TableSet tabs;
  tabs.n = n_tables;
  for (int i = 0; i < n_tables; ++i) {
    if (!tables_dev[i]) return fail(ISD_EINVAL, "NULL table %d", i);
    tabs.t[i] = reinterpret_cast<const unsigned long long*>(tables_dev[i]);
  }
  const int r = launch_thermo_set(
      tabs, reinterpret_cast<unsigned long long*>(sum_dev), n_spins, n_bonds,
      energy_scale, fields_dev, n_fields, temps_dev, n_temps, out_dev, stream);
  if (r < 0) return cuda_fail((cudaError_t)(-r), "k2 gather launch");
  bump_launches((uint64_t)r);
  return ISD_OK;
}

int isd_naive_enumerate(uint32_t n_spins, const uint32_t* bit_of_slot,
                        uint32_t n_bonds, const uint32_t* bond_slots,
                        const int32_t* bond_sign, int coupling_sign,
                        uint64_t start, uint64_t end, int device,
                        uint64_t* counts_host) {
  if (!bit_of_slot || (n_bonds && (!bond_slots || !bond_sign)) ||
      !counts_host)
    return fail(ISD_EINVAL, "NULL buffer");
  if (n_spins < 1 || n_spins > ISD_MAX_SPINS || n_bonds > 3 * ISD_MAX_SPINS)
    return fail(ISD_EINVAL, "bad lattice N=%u B=%u", n_spins, n_bonds);
  if (!(start <= end && end <= (1ull << n_spins)))
    return fail(ISD_EINVAL, "range [%llu, %llu) invalid for 2^%u configurations",
                (unsigned long long)start, (unsigned long long)end, n_spins);
  DeviceGuard guard;
  DevState* s = nullptr;
  std::unique_lock<std::mutex> lock;
  int rc = get_dev(device, &s, &lock);
  if (rc) return rc;
  const size_t bytes = (size_t)(n_spins + 1) * (n_bonds + 1) * 8;
  rc = ensure_buffer(&s->d_counts, &s->d_counts_bytes, bytes,
                     "cudaMalloc(counts)");
  if (rc) return rc;
  cudaError_t e = cudaMemsetAsync(s->d_counts, 0, bytes, s->stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  std::string why;
  const int r = naive_enumerate(n_spins, bit_of_slot, n_bonds, bond_slots,
                                bond_sign, coupling_sign, start, end,
                                s->d_counts, s->sm_count, s->stream, &why);
  if (r < 0) {
    if (!why.empty()) return fail(ISD_EINVAL, "%s", why.c_str());
    return cuda_fail((cudaError_t)(-r), "k5_naive launch");
  }
  bump_launches((uint64_t)r);
  void* stage = nullptr;
  rc = stage_buffer(s, bytes, &stage);
  if (rc) return rc;
  e = cudaMemcpyAsync(stage, s->d_counts, bytes, cudaMemcpyDeviceToHost,
                      s->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return cuda_fail(e, "naive enumeration");
  std::memcpy(counts_host, stage, bytes);
  return ISD_OK;
}

int isd_mirror_async(uint64_t* counts_dev, uint32_t n_spins, uint32_t n_bonds,
                     void* stream) {
  if (!counts_dev || n_spins < 1 || n_spins > ISD_MAX_SPINS ||
      n_bonds > 3 * ISD_MAX_SPINS)
    return fail(ISD_EINVAL, "bad table N=%u B=%u", n_spins, n_bonds);
  int r = launch_mirror(reinterpret_cast<unsigned long long*>(counts_dev),
                        n_spins, n_bonds, stream);
  if (r < 0) return cuda_fail((cudaError_t)(-r), "k3_mirror launch");
  bump_launches((uint64_t)r);
  return ISD_OK;
}

int isd_thermo_async(const uint64_t* counts_dev, uint32_t n_spins,
                     uint32_t n_bonds, double energy_scale,
                     const double* fields_dev, int n_fields,
                     const double* temps_dev, int n_temps, double* out_dev,
                     void* stream) {
  if (n_spins < 1 || n_spins > ISD_MAX_SPINS || n_bonds > 3 * ISD_MAX_SPINS)
    return fail(ISD_EINVAL, "bad table shape N=%u B=%u", n_spins, n_bonds);
  if (n_fields < 0 || n_temps < 0)
    return fail(ISD_EINVAL, "negative grid size");
  if (!(energy_scale > 0)) return fail(ISD_EINVAL, "energy_scale must be > 0");
  if (!counts_dev || (n_fields * n_temps > 0 &&
                      (!fields_dev || !temps_dev || !out_dev)))
    return fail(ISD_EINVAL, "NULL buffer");
  int r = launch_thermo(reinterpret_cast<const unsigned long long*>(counts_dev),
                        n_spins, n_bonds, energy_scale, fields_dev, n_fields,
                        temps_dev, n_temps, out_dev, stream);
  if (r < 0) return cuda_fail((cudaError_t)(-r), "k2_thermo launch");
  bump_launches((uint64_t)r);
  return ISD_OK;
}

int isd_thermo(const uint64_t* counts_host, uint32_t n_spins, uint32_t n_bonds,
               double energy_scale, const double* fields, int n_fields,
               const double* temps, int n_temps, int device, double* out_host,
               double* device_ms) {
  if (n_spins < 1 || n_spins > ISD_MAX_SPINS || n_bonds > 3 * ISD_MAX_SPINS)
    return fail(ISD_EINVAL, "bad table shape N=%u B=%u", n_spins, n_bonds);
  if (!counts_host || !fields || !temps || !out_host)
    return fail(ISD_EINVAL, "NULL buffer");
  if (n_fields < 0 || n_temps < 0)
    return fail(ISD_EINVAL, "negative grid size");
  DeviceGuard guard;
  DevState* s = nullptr;
  std::unique_lock<std::mutex> lock;
  int rc = get_dev(device, &s, &lock);
  if (rc) return rc;
  // one block, host and device alike: [table | fields | temps | results]
  const size_t tbytes = (size_t)(n_spins + 1) * (n_bonds + 1) * 8;
  const size_t npts = (size_t)n_fields * n_temps;
  const size_t in_bytes = tbytes + (size_t)(n_fields + n_temps) * 8;
  const size_t out_bytes = npts * ISD_THERMO_FIELDS * 8;
  if (s->d_buf_bytes < in_bytes + out_bytes) {
    if (s->d_buf) cudaFree(s->d_buf);
    s->d_buf = nullptr;
    s->d_buf_bytes = 0;
    cudaError_t e = cudaMalloc(&s->d_buf, in_bytes + out_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(thermo)");
    s->d_buf_bytes = in_bytes + out_bytes;
  }
  void* stage = nullptr;
  rc = stage_buffer(s, in_bytes + out_bytes, &stage);
  if (rc) return rc;
  char* h = static_cast<char*>(stage);
  std::memcpy(h, counts_host, tbytes);
  std::memcpy(h + tbytes, fields, (size_t)n_fields * 8);
  std::memcpy(h + tbytes + (size_t)n_fields * 8, temps, (size_t)n_temps * 8);
  char* d = reinterpret_cast<char*>(s->d_buf);
  const uint64_t* d_c = reinterpret_cast<const uint64_t*>(d);
  const double* d_f = reinterpret_cast<const double*>(d + tbytes);
  const double* d_t = d_f + n_fields;
  double* d_o = reinterpret_cast<double*>(d + in_bytes);
  cudaStream_t st = s->stream;
  cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, st);
  cudaEventRecord(s->ev0, st);
  rc = isd_thermo_async(d_c, n_spins, n_bonds, energy_scale, d_f, n_fields,
                        d_t, n_temps, d_o, st);
  if (rc) return rc;
  cudaEventRecord(s->ev1, st);
  cudaError_t e = cudaMemcpyAsync(h + in_bytes, d_o, out_bytes,
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "thermo kernel");
  std::memcpy(out_host, h + in_bytes, out_bytes);
  if (device_ms) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s->ev0, s->ev1);
    *device_ms = ms;
  }
  return ISD_OK;
}

int isd_calibrate(int device, int which, double* lanes_per_clk_sm,
                  double* sm_mhz) {
  DeviceGuard guard;
  DevState* s = nullptr;
  std::unique_lock<std::mutex> lock;
  int rc = get_dev(device, &s, &lock);
  if (rc) return rc;
  if (which < 0 || which > 12) return fail(ISD_EINVAL, "unknown probe %d", which);
  double lanes = 0, mhz = 0;
  int r = run_calibration(which, s->sm_count, &lanes, &mhz);
  if (r < 0) return cuda_fail((cudaError_t)(-r), "k0 calibration");
  if (lanes_per_clk_sm) *lanes_per_clk_sm = lanes;
  if (sm_mhz) *sm_mhz = mhz;
  return ISD_OK;
}

int isd_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int isd_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) !=
      cudaSuccess)
    return fail(ISD_ENODEV, "no device %d", device);
  return v;
}

int isd_set_knob(const char* name, const char* value) {
  if (!name || !knob_known(name))
    return fail(ISD_EINVAL, "unknown knob %s", name ? name : "(null)");
  forget_prepared();
  return set_knob(name, value);
}

int isd_clear_knobs(void) {
  forget_prepared();
  clear_knobs();
  return ISD_OK;
}

int isd_set_cache_dirs(const char* dirs) {
  set_cache_dirs(dirs ? dirs : "");
  return ISD_OK;
}

const char* isd_build_id(void) { return build_id(); }

const char* isd_last_error(void) { return g_err.c_str(); }
const char* isd_kernel_info(void) { return g_kernel_info.c_str(); }
const char* isd_version(void) { return "isingdos-b200 0.1.0 (sm_100a)"; }
int isd_abi_version(void) { return ISD_ABI_VERSION; }
uint64_t isd_launch_count(void) { return g_launches.load(); }

}  // extern "C"
