// Host engine: device residency of the model tables, the value-iteration
// driver (run_value_iteration, vi.hpp:162-291), single-sweep entry points
// and the PVI1 checkpoint format (checkpoint.cpp).  The driver keeps V and
// its history on the device; per sweep the host reads back one 32-byte
// statistics record (max/min of the convergence statistic and the first
// non-finite state), so the only host round trip is that flag.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <exception>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "engine.hpp"
#include "vi_kernels.cuh"

namespace pvi_b200 {

// ---------------------------------------------------------------------------
// Device residency

namespace {

template <typename U>
const U* upload(DeviceCopy& dc, const std::vector<U>& host) {
  if (host.empty()) return nullptr;
  void* p = nullptr;
  PVI_CUDA(cudaMalloc(&p, host.size() * sizeof(U)));
  upload_bytes(p, host.data(), host.size() * sizeof(U));
  dc.allocations.push_back(p);
  return static_cast<const U*>(p);
}

}  // namespace

// Device buffers reused across pvi_vi_backup / pvi_q_rows calls on one
// model, so a serving caller pays for the copies and the sweep only.
struct Workspace {
  static constexpr int kChunkEvents = 16;
  std::mutex mu;
  Scratch scratch;  // sweep scratch (partials, factored tables)
  Scratch io;       // 0: V, 1: V' slice, 2: argmax slice, 3: Q rows
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;  // device-to-host results of finished chunks
  cudaStream_t copy2 = nullptr;  // the argmax half of them (a second copy queue)
  cudaStream_t up = nullptr;    // host-to-device pieces (the other PCIe direction)
  cudaStream_t s2[2] = {};      // stage 2 of consecutive x_3 pairs, overlapping
  cudaEvent_t done[kChunkEvents] = {};
  cudaEvent_t ev[4 * kChunkEvents] = {};
  Workspace() {
    // `stream` carries the pipelined backup's stage-1 pieces: highest
    // priority, so they are scheduled ahead of the stage-2 grids they feed
    int least = 0, greatest = 0;
    PVI_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    PVI_CUDA(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, greatest));
    PVI_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    PVI_CUDA(cudaStreamCreateWithFlags(&copy2, cudaStreamNonBlocking));
    PVI_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    for (auto& x : s2) PVI_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    for (auto& e : done) PVI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : ev) PVI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~Workspace() {
    for (auto& e : done)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& x : s2)
      if (x) cudaStreamDestroy(x);
    if (copy) cudaStreamDestroy(copy);
    if (copy2) cudaStreamDestroy(copy2);
    if (up) cudaStreamDestroy(up);
    if (stream) cudaStreamDestroy(stream);
  }
};

Model::~Model() {
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto& kv : dev) {
    cudaSetDevice(kv.first);
    delete static_cast<Workspace*>(kv.second->workspace);
    for (void* p : kv.second->allocations) cudaFree(p);
  }
  if (prev >= 0) cudaSetDevice(prev);
}

Workspace& workspace(const Model& m, int device) {
  DeviceCopy& dc = m.device_copy(device);
  std::lock_guard<std::mutex> lock(m.dev_mutex);
  if (!dc.workspace) dc.workspace = new Workspace();
  return *static_cast<Workspace*>(dc.workspace);
}

const DevModel& Model::device_view(int device) const {
  std::lock_guard<std::mutex> lock(dev_mutex);
  auto it = dev.find(device);
  if (it != dev.end()) return it->second->dm;
  auto dc = std::make_unique<DeviceCopy>();
  DevModel& d = dc->dm;
  d.scenario = scenario;
  d.n_digits = static_cast<int>(space.radix.size());
  d.n_states = space.count;
  d.n_actions = n_actions;
  for (int i = 0; i < d.n_digits; ++i) {
    d.weight[i] = space.weight[i];
    d.radix[i] = space.radix[i];
  }
  switch (scenario) {
    case PVI_SCENARIO_A:
      d.a_m = pa.useful_life;
      d.a_lead = pa.lead_time;
      d.a_lifo = pa.issuing != 0;
      d.a_max_order = pa.max_order;
      d.a_dmax = pa.max_demand;
      d.a_cv = pa.unit_cost;
      d.a_ch = pa.holding_cost;
      d.a_cs = pa.shortage_cost;
      d.a_cw = pa.wastage_cost;
      d.a_pmf = upload(*dc, a_pmf);
      d.a_cdf = upload(*dc, a_cdf);
      d.a_guide = upload(*dc, cdf_guide(a_cdf.data(), pa.max_demand + 1, kGuide));
      break;
    case PVI_SCENARIO_B:
      d.b_m = pb.useful_life;
      d.b_na = b_na;
      d.b_nb = b_nb;
      d.b_cap_a = b_cap_a;
      d.b_cap_b = b_cap_b;
      d.b_dn = b_dmax + 1;
      d.b_len_a = static_cast<int>(b_pmf_a.size());
      d.b_len_b = static_cast<int>(b_pmf_b.size());
      d.b_cva = pb.unit_cost_a;
      d.b_cvb = pb.unit_cost_b;
      d.b_cra = pb.revenue_a;
      d.b_crb = pb.revenue_b;
      d.b_rho = pb.substitution_prob;
      d.b_mu_a = pb.demand_mean_a;
      d.b_mu_b = pb.demand_mean_b;
      d.b_pmf_a = upload(*dc, b_pmf_a);
      d.b_pmf_b = upload(*dc, b_pmf_b);
      d.b_sf_a = upload(*dc, b_sf_a);
      d.b_sf_b = upload(*dc, b_sf_b);
      d.b_pz = upload(*dc, b_pz);
      d.b_pz_cum = upload(*dc, b_pz_cum);
      d.b_cdf_a = upload(*dc, b_cdf_a);
      d.b_cdf_b = upload(*dc, b_cdf_b);
      d.b_guide_a = upload(*dc, cdf_guide(b_cdf_a.data(), static_cast<int>(b_cdf_a.size()), kGuide));
      d.b_guide_b = upload(*dc, cdf_guide(b_cdf_b.data(), static_cast<int>(b_cdf_b.size()), kGuide));
      // trials = demand_b - fill_b <= |support of demand_b| - 1
      d.b_binom_t = static_cast<int>(b_pmf_b.size()) - 1;
      d.b_binom_cum = nullptr;
      d.b_binom_guide = nullptr;
      if (pb.substitution_prob > 0.0 && pb.substitution_prob < 1.0) {
        const auto cum = binomial_cum_table(d.b_binom_t, pb.substitution_prob);
        d.b_binom_cum = upload(*dc, cum);
        d.b_binom_guide = upload(*dc, binomial_guide_table(cum, d.b_binom_t, kBinGuide));
      }
      d.b_lane_order = upload(*dc, b_lane_order);
      d.b_tile = static_cast<int>(b_lane_order.size());
      break;
    case PVI_SCENARIO_C:
      d.c_m = pc.useful_life;
      d.c_max_order = pc.max_order;
      d.c_dmax = pc.max_demand;
      d.c_n_comp = c_n_comp;
      d.c_cf = pc.fixed_order_cost;
      d.c_ch = pc.holding_cost;
      d.c_cs = pc.shortage_cost;
      d.c_cw = pc.wastage_cost;
      d.c_pmf = upload(*dc, c_pmf);
      d.c_cdf = upload(*dc, c_cdf);
      {
        const int dn = pc.max_demand + 1;
        std::vector<double> pd(7, 0.0);  // the kernels' former per-CTA loop, same order
        for (int t = 0; t < 7; ++t)
          for (int dd = 0; dd < dn; ++dd) pd[t] += c_pmf[static_cast<std::size_t>(t) * dn + dd];
        d.c_pd = upload(*dc, pd);
        std::vector<std::int32_t> g;
        for (int t = 0; t < 7; ++t) {
          const auto gt = cdf_guide(c_cdf.data() + static_cast<std::size_t>(t) * dn, dn, kGuide);
          g.insert(g.end(), gt.begin(), gt.end());
        }
        d.c_guide = upload(*dc, g);
        std::vector<double> cum;
        std::vector<std::int32_t> off;
        c_receipt_tables(c_receipt.data(), pc.max_order, pc.useful_life, cum, off);
        d.c_rcpt_cum = upload(*dc, cum);
        d.c_rcpt_off = upload(*dc, off);
        // each (a, k) table's guide rows at a parallel offset
        std::vector<std::int32_t> goff(off.size(), -1), guide;
        for (std::size_t i = 0; i < off.size(); ++i) {
          if (off[i] < 0) continue;
          const int a = static_cast<int>(i / (pc.useful_life - 1));
          const std::vector<double> tab(cum.begin() + off[i],
                                        cum.begin() + off[i] + static_cast<std::ptrdiff_t>(a + 1) * (a + 2) / 2);
          const auto gt = binomial_guide_table(tab, a, kBinGuide);
          goff[i] = static_cast<std::int32_t>(guide.size());
          guide.insert(guide.end(), gt.begin(), gt.end());
        }
        d.c_rcpt_goff = upload(*dc, goff);
        d.c_rcpt_guide = guide.empty() ? nullptr : upload(*dc, guide);
      }
      d.c_comp = upload(*dc, c_comp);
      d.c_ids = upload(*dc, c_ids);
      d.c_probs = upload(*dc, c_probs);
      d.c_offsets = upload(*dc, c_offsets);
      d.c_receipt = upload(*dc, c_receipt);
      d.c_exogenous = c_exogenous ? 1 : 0;
      d.c_binom = c_binom.empty() ? nullptr : upload(*dc, c_binom);
      d.c_frag = nullptr;
      d.c_gband = d.c_ra = d.c_cwt = nullptr;
      if (pc.max_order == 20 && pc.max_demand == 20) {
        constexpr int DN = 21, CAP = 20, NT = 2 * DN - 1, NF = 3 * 7 * 32;
        std::vector<double> band(7 * static_cast<std::size_t>(NF), 0.0);
        for (int t = 0; t < 7; ++t)
          for (int e = 0; e < NF; ++e) {
            const int i = e / (7 * 32), j = (e / 32) % 7, ln = e % 32;
            const int row = 8 * i + (ln >> 2), col = 4 * (2 * i + j) + (ln & 3);  // T[z_1][t]
            const int dd = row - col + CAP;
            band[static_cast<std::size_t>(t) * NF + e] =
                (row < DN && col < NT && dd >= 0 && dd <= CAP) ? c_pmf[static_cast<std::size_t>(t) * DN + dd] : 0.0;
          }
        const int nra = pc.useful_life * (DN - 1) + DN;
        std::vector<double> ra(nra), cw(DN);
        for (int i = 0; i < nra; ++i) {
          const int x = i - (DN - 1);
          ra[i] = -pc.holding_cost * static_cast<double>(std::max(x, 0)) -
                  pc.shortage_cost * static_cast<double>(std::max(-x, 0));
        }
        for (int i = 0; i < DN; ++i) cw[i] = pc.wastage_cost * static_cast<double>(i);
        d.c_gband = upload(*dc, band);
        d.c_ra = upload(*dc, ra);
        d.c_cwt = upload(*dc, cw);
      }
      if (!c_binom.empty() && !c_exogenous && pc.max_order == 20) {
        // [t][s][lane] = L[8 t + lane / 4][4 s + lane % 4], L[b][b'] =
        // Bin(b - b'; b, q_k(a)) for b' <= b < a + 1 (c_pass_fragments' layout)
        constexpr int R = 21, NF = 3 * 6 * 32;
        const int life = pc.useful_life;
        std::vector<double> fr(static_cast<std::size_t>(R) * (life - 1) * NF, 0.0);
        for (int a = 0; a < R; ++a)
          for (int k = 1; k <= life - 1; ++k) {
            const double* bt = &c_binom[(static_cast<std::size_t>(a) * (life - 1) + (k - 1)) * R * R];
            double* out = &fr[(static_cast<std::size_t>(a) * (life - 1) + (k - 1)) * NF];
            for (int e = 0; e < NF; ++e) {
              const int t = e / (6 * 32), sk = (e / 32) % 6, ln = e & 31;
              const int b = 8 * t + (ln >> 2), bp = 4 * sk + (ln & 3);
              out[e] = (bp <= b && b < a + 1) ? bt[b * R + (b - bp)] : 0.0;
            }
          }
        d.c_frag = upload(*dc, fr);
      }
      break;
    default:
      d.t_outcomes = n_outcomes;
      d.t_next = upload(*dc, t_next);
      d.t_reward = upload(*dc, t_reward);
      d.t_prob = upload(*dc, t_prob);
      break;
  }
  const DevModel& out = dc->dm;
  dev.emplace(device, std::move(dc));
  return out;
}

DeviceCopy& Model::device_copy(int device) const {
  device_view(device);
  std::lock_guard<std::mutex> lock(dev_mutex);
  return *dev.at(device);
}

int select_device(int requested) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(PVI_ERR_DEVICE, "no CUDA device available (pvi_b200 has no CPU fallback)");
  }
  int dev = requested;
  if (dev < 0) PVI_CUDA(cudaGetDevice(&dev));
  if (dev >= count) fail(PVI_ERR_DEVICE, "CUDA device ordinal out of range");
  PVI_CUDA(cudaSetDevice(dev));
  return dev;
}

// ---------------------------------------------------------------------------
// Small RAII helpers

struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  explicit DevBuf(std::size_t bytes) {
    if (bytes) PVI_CUDA(cudaMalloc(&p, bytes));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename U>
  U* as() const {
    return static_cast<U*>(p);
  }
};

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { PVI_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s) cudaStreamDestroy(s);
  }
};

// Pinned 32-byte statistics record, one per host thread (cudaMallocHost is
// a driver call of ~ms; a solve should not pay it each time).
struct PinnedStats {
  SweepStats* h = nullptr;
  PinnedStats() {
    static thread_local SweepStats* cached = nullptr;
    if (!cached) PVI_CUDA(cudaMallocHost(&cached, sizeof(SweepStats)));
    h = cached;
  }
};

// ---------------------------------------------------------------------------
// Checkpoints (checkpoint.hpp:24-35): "PVI1" | iteration u64 LE |
// fingerprint[32] | count u64 LE | count x f64 LE; temp file + rename.

void save_checkpoint(const std::string& path, const double* values, std::uint64_t count,
                     std::uint64_t iteration, const std::uint8_t fp[32]) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    if (!out) fail(PVI_ERR_IO, "cannot open checkpoint file for writing: " + tmp);
    unsigned char header[52];
    std::memcpy(header, "PVI1", 4);
    for (int i = 0; i < 8; ++i) header[4 + i] = static_cast<unsigned char>(iteration >> (8 * i));
    std::memcpy(header + 12, fp, 32);
    for (int i = 0; i < 8; ++i) header[44 + i] = static_cast<unsigned char>(count >> (8 * i));
    out.write(reinterpret_cast<const char*>(header), sizeof(header));
    // x86-64 and the device are little-endian: the payload is the raw bits.
    out.write(reinterpret_cast<const char*>(values), static_cast<std::streamsize>(count * 8));
    if (!out) fail(PVI_ERR_IO, "failed writing checkpoint: " + tmp);
  }
  std::error_code ec;
  std::filesystem::rename(tmp, path, ec);
  if (ec) fail(PVI_ERR_IO, "failed to move checkpoint into place: " + ec.message());
}

void load_checkpoint(const std::string& path, const std::uint8_t* expected, double* values,
                     std::uint64_t capacity, std::uint64_t* count, std::uint64_t* iteration,
                     std::uint8_t fp[32]) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(PVI_ERR_IO, "cannot open checkpoint file: " + path);
  unsigned char header[52];
  in.read(reinterpret_cast<char*>(header), sizeof(header));
  if (!in || std::memcmp(header, "PVI1", 4) != 0)
    fail(PVI_ERR_FORMAT, "not a checkpoint file (bad magic): " + path);
  std::uint64_t it = 0, n = 0;
  for (int i = 0; i < 8; ++i) it |= static_cast<std::uint64_t>(header[4 + i]) << (8 * i);
  for (int i = 0; i < 8; ++i) n |= static_cast<std::uint64_t>(header[44 + i]) << (8 * i);
  if (fp) std::memcpy(fp, header + 12, 32);
  if (count) *count = n;
  if (iteration) *iteration = it;
  if (expected && std::memcmp(expected, header + 12, 32) != 0) {
    fail(PVI_ERR_FINGERPRINT, "checkpoint fingerprint " + hex32(header + 12) +
                                  " does not match model fingerprint " + hex32(expected));
  }
  if (!values) {
    // Still validate the payload length.
    in.seekg(0, std::ios::end);
    const auto size = static_cast<std::uint64_t>(in.tellg());
    if (size < 52 + 8 * n) fail(PVI_ERR_FORMAT, "checkpoint truncated: " + path);
    return;
  }
  if (n > capacity) fail(PVI_ERR_FORMAT, "checkpoint larger than the destination buffer");
  in.read(reinterpret_cast<char*>(values), static_cast<std::streamsize>(n * 8));
  if (!in) fail(PVI_ERR_FORMAT, "checkpoint truncated: " + path);
}

// Asynchronous PVI1 writer: the sweep stream widens V into a
// device slot and copies it into one of two pinned host slots; a worker
// thread waits on the copy's event and writes the file (temp + rename)
// while the next sweeps run.  Writes stay in iteration order; the first I/O
// error is rethrown at the next submit or at finish().
class AsyncCheckpointer {
 public:
  AsyncCheckpointer(std::string path, std::uint64_t n, const std::uint8_t fp[32])
      : path_(std::move(path)), n_(n) {
    std::memcpy(fp_, fp, 32);
    PVI_CUDA(cudaGetDevice(&device_));
    for (auto& s : slots_) {
      PVI_CUDA(cudaMallocHost(&s.host, n * sizeof(double)));
      PVI_CUDA(cudaMalloc(&s.dev, n * sizeof(double)));
      PVI_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    }
    worker_ = std::thread([this] { run(); });
  }
  ~AsyncCheckpointer() {
    try {
      finish();
    } catch (...) {
    }
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (worker_.joinable()) worker_.join();
    for (auto& s : slots_) {
      if (s.host) cudaFreeHost(s.host);
      if (s.dev) cudaFree(s.dev);
      if (s.done) cudaEventDestroy(s.done);
    }
  }
  double* acquire() {
    std::unique_lock<std::mutex> lock(mu_);
    cur_ = (cur_ + 1) % 2;
    cv_.wait(lock, [&] { return !slots_[cur_].busy || error_; });
    if (error_) std::rethrow_exception(error_);
    slots_[cur_].busy = true;
    return slots_[cur_].host;
  }
  double* device_slot() { return slots_[cur_].dev; }
  void submit(std::uint64_t iteration, cudaStream_t stream) {
    PVI_CUDA(cudaEventRecord(slots_[cur_].done, stream));
    {
      std::lock_guard<std::mutex> lock(mu_);
      queue_.push_back({cur_, iteration});
    }
    cv_.notify_all();
  }
  void finish() {
    std::unique_lock<std::mutex> lock(mu_);
    cv_.wait(lock, [&] { return (queue_.empty() && !slots_[0].busy && !slots_[1].busy) || error_; });
    if (error_) {
      auto e = error_;
      error_ = nullptr;
      std::rethrow_exception(e);
    }
  }

 private:
  struct Slot {
    double* host = nullptr;
    double* dev = nullptr;
    cudaEvent_t done = nullptr;
    bool busy = false;
  };
  void run() {
    cudaSetDevice(device_);
    for (;;) {
      std::pair<int, std::uint64_t> job;
      {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] { return stop_ || !queue_.empty(); });
        if (queue_.empty()) return;
        job = queue_.front();
        queue_.pop_front();
      }
      try {
        PVI_CUDA(cudaEventSynchronize(slots_[job.first].done));
        save_checkpoint(path_, slots_[job.first].host, n_, job.second, fp_);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu_);
        if (!error_) error_ = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lock(mu_);
        slots_[job.first].busy = false;
      }
      cv_.notify_all();
    }
  }
  std::string path_;
  std::uint64_t n_;
  std::uint8_t fp_[32];
  int device_ = 0;
  Slot slots_[2];
  int cur_ = 1;
  std::thread worker_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::pair<int, std::uint64_t>> queue_;
  bool stop_ = false;
  std::exception_ptr error_;
};

std::string hex32(const std::uint8_t* fp) {
  static const char* digits = "0123456789abcdef";
  std::string s;
  for (int i = 0; i < 32; ++i) {
    s.push_back(digits[fp[i] >> 4]);
    s.push_back(digits[fp[i] & 15]);
  }
  return s;
}

// ---------------------------------------------------------------------------
// Initial values (vi.hpp:197-200): f64 on the device.

void initial_values_device(const Model& m, const DevModel& dm, double* out, cudaStream_t stream) {
  const std::uint64_t n = m.space.count;
  switch (m.scenario) {
    case PVI_SCENARIO_B:
      launch_initial_b(dm, out, n, stream);
      break;
    case PVI_TABULAR:
      PVI_CUDA(cudaMemcpyAsync(out, m.t_initial.data(), n * 8, cudaMemcpyHostToDevice, stream));
      break;
    default:
      PVI_CUDA(cudaMemsetAsync(out, 0, n * 8, stream));
  }
}

void initial_values_host(const Model& m, double* out) {
  const int device = select_device(-1);
  const DevModel& dm = m.device_view(device);
  const std::uint64_t n = m.space.count;
  Stream stream;
  DevBuf d(n * sizeof(double));
  initial_values_device(m, dm, d.as<double>(), stream.s);
  PVI_CUDA(cudaMemcpyAsync(out, d.p, n * 8, cudaMemcpyDeviceToHost, stream.s));
  PVI_CUDA(cudaStreamSynchronize(stream.s));
}

// ---------------------------------------------------------------------------
// Value iteration driver (vi.hpp:162-291)

namespace {

// Device -> host copy into the caller's memory at pinned-copy speed.  A
// run_value_iteration caller (a std::vector, a numpy array) hands pageable
// memory, which the driver copies at ~21 GB/s through its own staging; here
// the copy goes through a pinned ring in 8 MB chunks, each landed chunk
// moved to the caller by a small persistent host pool while the next chunks
// are in flight (~45 GB/s measured on the B200 host, tools/pageable_probe.py).
// Pinned (page-locked or registered) destinations take one cudaMemcpyAsync.
class BounceCopier {
 public:
  static BounceCopier& get() {
    static BounceCopier b;
    return b;
  }
  void copy(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, dst) == cudaSuccess &&
                        (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged);
    cudaGetLastError();  // an unregistered pointer is not an error here
    if (pinned || bytes <= kChunk) {
      PVI_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
      PVI_CUDA(cudaStreamSynchronize(s));
      return;
    }
    std::lock_guard<std::mutex> lock(use_mu_);
    int device = 0;
    PVI_CUDA(cudaGetDevice(&device));
    if (device < 0 || device >= kMaxDevices) fail(PVI_ERR_DEVICE, "device ordinal out of range");
    Ring& rg = ring(device);  // events belong to the stream's device
    const std::size_t n_chunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](std::size_t i) {
      const std::size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
      PVI_CUDA(cudaMemcpyAsync(rg.buf[i % kSlots], static_cast<const char*>(src) + off, len,
                               cudaMemcpyDeviceToHost, s));
      PVI_CUDA(cudaEventRecord(rg.ev[i % kSlots], s));
    };
    for (std::size_t i = 0; i < std::min<std::size_t>(kSlots, n_chunks); ++i) issue(i);
    for (std::size_t i = 0; i < n_chunks; ++i) {
      PVI_CUDA(cudaEventSynchronize(rg.ev[i % kSlots]));
      const std::size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
      parallel_memcpy(static_cast<char*>(dst) + off, rg.buf[i % kSlots], len);
      if (i + kSlots < n_chunks) issue(i + kSlots);
    }
  }

 private:
  static constexpr std::size_t kChunk = 8u << 20;
  static constexpr int kSlots = 3, kThreads = 4;
  BounceCopier() {
    for (int t = 0; t < kThreads; ++t) pool_.emplace_back([this, t] { worker(t); });
  }
  ~BounceCopier() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& th : pool_) th.join();
  }
  struct Ring {
    char* buf[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
  };
  static constexpr int kMaxDevices = 64;
  Ring& ring(int device) {  // pinned (portable) slots and events of one device, made on first use
    Ring& rg = rings_[device];
    if (rg.buf[0]) return rg;
    for (int k = 0; k < kSlots; ++k) {
      PVI_CUDA(cudaHostAlloc(&rg.buf[k], kChunk, cudaHostAllocPortable));
      PVI_CUDA(cudaEventCreateWithFlags(&rg.ev[k], cudaEventDisableTiming));
    }
    return rg;
  }
  void parallel_memcpy(char* dst, const char* src, std::size_t len) {
    {
      std::lock_guard<std::mutex> l(mu_);
      job_dst_ = dst;
      job_src_ = src;
      job_len_ = len;
      pending_ = kThreads;
      ++gen_;
    }
    cv_.notify_all();
    std::unique_lock<std::mutex> l(mu_);
    done_cv_.wait(l, [&] { return pending_ == 0; });
  }
  void worker(int t) {
    std::uint64_t seen = 0;
    for (;;) {
      char* d;
      const char* sr;
      std::size_t len;
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        d = job_dst_;
        sr = job_src_;
        len = job_len_;
      }
      const std::size_t per = (len / kThreads + 63) & ~std::size_t(63);
      const std::size_t a = std::min(len, per * t), b = std::min(len, per * (t + 1));
      if (b > a) std::memcpy(d + a, sr + a, b - a);
      {
        std::lock_guard<std::mutex> l(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::mutex use_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> pool_;
  bool stop_ = false;
  std::uint64_t gen_ = 0;
  int pending_ = 0;
  char* job_dst_ = nullptr;
  const char* job_src_ = nullptr;
  std::size_t job_len_ = 0;
  Ring rings_[kMaxDevices];
};

bool evaluate_test(int test, double hi, double lo, double epsilon, std::uint64_t iteration) {
  switch (test) {
    case PVI_TEST_VALUE_SPAN:
      return std::max(0.0, hi) < epsilon;
    case PVI_TEST_CHANGE_SPAN:
      return hi - lo < epsilon;
    default:
      if (iteration < 7) return false;
      return hi - lo <= 2.0 * epsilon * std::min(std::abs(hi), std::abs(lo));
  }
}

// Graph-resident sweep loop.  The loop control of run_value_iteration
// (vi.hpp:220-265: divergence check, convergence test, iteration limit) is
// evaluated by a one-thread kernel after every sweep, which sets the
// condition of the CUDA graph's WHILE node, so a solve runs as ONE graph
// launch with no host round trip per sweep.  The value ring has two slots
// (value / change span), so the WHILE body holds two sweeps (b -> a, then
// a -> b inside an IF node the first decision also sets).
bool loop_trace() {
  static const bool on = [] {
    const char* e = std::getenv("PVI_LOOP_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}

// one slot of the device value ring (a view into one allocation)
struct RingSlot {
  void* p;
  template <typename U>
  U* as() const {
    return static_cast<U*>(p);
  }
};

struct LoopState {
  unsigned long long iteration;  // absolute sweep count
  unsigned long long limit;      // stop once iteration reaches it
  unsigned long long first_bad;  // first non-finite state, ~0 when none
  unsigned long long bad_iteration;
  double last_hi, last_lo;
  double epsilon;
  int test;                      // -1: no test (fixed iterations)
  int fixed;                     // fixed_iterations mode: reaching the limit converges
  int converged;
  int pad;
};

__device__ bool loop_decide(LoopState* ls, SweepStats* st) {
  LoopState s = *ls;
  s.iteration += 1;
  bool stop = false;
  if (st->first_bad != ~0ull) {
    s.first_bad = st->first_bad;
    s.bad_iteration = s.iteration;
    stop = true;
  } else {
    if (s.test >= 0) {
      const double hi = dkey_inv(st->max_key);
      const double lo = s.test == PVI_TEST_VALUE_SPAN ? 0.0 : dkey_inv(st->min_key);
      s.last_hi = hi;
      s.last_lo = lo;
      bool c;
      if (s.test == PVI_TEST_VALUE_SPAN) c = (0.0 < hi ? hi : 0.0) < s.epsilon;  // std::max(0.0, hi)
      else if (s.test == PVI_TEST_PERIODIC_SPAN)  // vi.hpp:150-156 (evaluate_test above)
        c = s.iteration >= 7 && hi - lo <= 2.0 * s.epsilon * fmin(fabs(hi), fabs(lo));
      else c = hi - lo < s.epsilon;  // change span
      s.converged = c ? 1 : 0;
      stop = c;
    }
    if (!stop && s.iteration >= s.limit) {
      if (s.fixed) s.converged = 1;
      stop = true;
    }
  }
  *ls = s;
  // reset the statistics for the next sweep (the graph's sweeps skip their
  // own k_init_stats launch: one kernel fewer per sweep)
  st->max_key = 0ull;
  st->min_key = ~0ull;
  st->first_bad = ~0ull;
  st->pad = 0;
  return stop;
}

__global__ void k_loop_decide(LoopState* ls, SweepStats* st, cudaGraphConditionalHandle h_while,
                              cudaGraphConditionalHandle h_if, int set_if) {
  const bool stop = loop_decide(ls, st);
  cudaGraphSetConditional(h_while, stop ? 0u : 1u);
  if (set_if) cudaGraphSetConditional(h_if, stop ? 0u : 1u);
}

// Eight-slot ring (periodic span): the WHILE body is a chain of eight IF
// nodes, one per ring phase; IF k sweeps into slot k of the rotation, then
// clears its own condition and arms IF k+1 (IF 0 in the next iteration).
__global__ void k_loop_decide_phase(LoopState* ls, SweepStats* st, cudaGraphConditionalHandle h_while,
                                    cudaGraphConditionalHandle h_self, cudaGraphConditionalHandle h_next) {
  const bool stop = loop_decide(ls, st);
  cudaGraphSetConditional(h_while, stop ? 0u : 1u);
  cudaGraphSetConditional(h_self, 0u);
  cudaGraphSetConditional(h_next, stop ? 0u : 1u);
}

// Persisting L2 window over [base, base + bytes) for kernels launched on
// `stream` (and captured from it): the value ring stays resident in L2
// while the sweeps gather from it.  Returns the window size (0: none).
std::size_t set_l2_window(cudaStream_t stream, const void* base, std::size_t bytes, int device,
                          double* hit_ratio) {
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
  if (max_persist <= 0 || max_window <= 0 || bytes == 0) return 0;
  const std::size_t win = std::min<std::size_t>(bytes, static_cast<std::size_t>(max_window));
  const std::size_t persist = std::min<std::size_t>(win, static_cast<std::size_t>(max_persist));
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaStreamAttrValue attr = {};
  attr.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  attr.accessPolicyWindow.num_bytes = win;
  attr.accessPolicyWindow.hitRatio = static_cast<float>(std::min(1.0, static_cast<double>(persist) / win));
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &attr) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  *hit_ratio = attr.accessPolicyWindow.hitRatio;
  return win;
}

void clear_l2_window(cudaStream_t stream) {
  cudaStreamAttrValue attr = {};
  attr.accessPolicyWindow.num_bytes = 0;
  cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &attr);
  cudaCtxResetPersistingL2Cache();
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  cudaGetLastError();
}

template <typename T>
void solve_impl(const Model& m, const pvi_vi_config& cfg, const double* resume_values,
                std::uint64_t resume_iteration, const std::uint8_t* resume_fp, double* out_values,
                std::uint32_t* out_policy, pvi_vi_stats* stats) {
  const auto t_start = std::chrono::steady_clock::now();
  const std::uint64_t n = m.space.count;
  if (n > cfg.max_states)
    fail(PVI_ERR_CAPACITY, "value iteration requires " + std::to_string(n) +
                               " states, exceeding the configured capacity of " +
                               std::to_string(cfg.max_states), n);
  if (n == 0) fail(PVI_ERR_PARAMETER, "value iteration: empty state space");
  const double gamma = cfg.has_gamma ? cfg.gamma : m.gamma;
  const int test = cfg.convergence_test >= 0 ? cfg.convergence_test : m.default_test;
  const int algo = cfg.algorithm >= 0 ? cfg.algorithm : m.algorithm;
  std::uint8_t fp[32];
  sha256(m.fingerprint.data(), m.fingerprint.size(), fp);

  const int device = select_device(cfg.device);
  const DevModel& dm = m.device_view(device);
  Stream stream;
  // sweep scratch (GB-scale for B: partials, factored W) reused across calls
  Workspace& ws = workspace(m, device);
  std::lock_guard<std::mutex> ws_lock(ws.mu);
  Scratch& scratch = ws.scratch;
  PinnedStats pstats;
  PoolBuf dstats(sizeof(SweepStats), stream.s);

  const int hist_cap = test == PVI_TEST_PERIODIC_SPAN ? 8 : 2;
  // the value ring is one allocation, so one L2 window covers every slot
  PoolBuf ring_mem(static_cast<std::size_t>(hist_cap) * n * sizeof(T), stream.s);
  std::vector<std::unique_ptr<RingSlot>> ring;
  for (int i = 0; i < hist_cap; ++i)
    ring.push_back(std::make_unique<RingSlot>(RingSlot{ring_mem.as<T>() + static_cast<std::size_t>(i) * n}));
  double l2_ratio = 0.0;
  const std::size_t l2_bytes =
      // auto: on for the exact kernels (their gathers hit the ring); off for
      // the factored sweeps, whose traffic is the W / G tables: a window over
      // the ring costs them L2 (tools/loop_ab.py on a B200: b/m3/exp1 solve
      // 78.5 -> 84.7 ms, c/m5/exp2 190 -> 225 ms with the window)
      (cfg.l2_persist == 0 || (cfg.l2_persist < 0 && algo == PVI_ALGO_FACTORED)) ? 0
                          : set_l2_window(stream.s, ring_mem.p, static_cast<std::size_t>(hist_cap) * n * sizeof(T),
                                          device, &l2_ratio);
  struct L2Reset {
    cudaStream_t s;
    bool on;
    ~L2Reset() {
      if (on) clear_l2_window(s);
    }
  } l2_reset{stream.s, l2_bytes > 0};
  std::vector<int> order;  // slots oldest..newest
  std::uint64_t iteration = 0;
  {
    PoolBuf v0(n * sizeof(double), stream.s);
    if (resume_values) {
      if (resume_fp && std::memcmp(resume_fp, fp, 32) != 0)
        fail(PVI_ERR_FINGERPRINT, "resume checkpoint fingerprint " + hex32(resume_fp) +
                                      " does not match model fingerprint " + hex32(fp));
      PVI_CUDA(cudaMemcpyAsync(v0.p, resume_values, n * 8, cudaMemcpyHostToDevice, stream.s));
      iteration = resume_iteration;
    } else {
      initial_values_device(m, dm, v0.as<double>(), stream.s);
    }
    launch_cast_from_f64<T>(v0.as<double>(), ring[0]->as<T>(), n, stream.s);
    order.push_back(0);
  }

  const bool ckpt = cfg.checkpoint_every > 0 && cfg.checkpoint_path && cfg.checkpoint_path[0];
  std::unique_ptr<AsyncCheckpointer> writer;
  if (ckpt) writer = std::make_unique<AsyncCheckpointer>(cfg.checkpoint_path, n, fp);
  auto write_checkpoint = [&](const T* dv, std::uint64_t iter) {
    if (!ckpt) return;
    double* wide = writer->acquire();  // waits only if both slots are still in flight
    launch_widen<T>(dv, writer->device_slot(), n, stream.s);
    PVI_CUDA(cudaMemcpyAsync(wide, writer->device_slot(), n * 8, cudaMemcpyDeviceToHost, stream.s));
    writer->submit(iter, stream.s);  // the file write overlaps the next sweeps
  };
  if (ckpt && !resume_values) write_checkpoint(ring[order.back()]->as<T>(), iteration);

  cudaEvent_t ev0, ev1;
  PVI_CUDA(cudaEventCreate(&ev0));
  PVI_CUDA(cudaEventCreate(&ev1));
  double sweep_ms = 0.0;
  std::uint64_t sweeps = 0;
  double last_hi = 0.0, last_lo = 0.0;

  bool converged = false;
  const std::uint64_t start_iteration = iteration;
  // graph-resident loop: two-vector tests, no checkpoint inside the loop,
  // not while the bench's per-launch profiler records events
  const bool graph_possible = !ckpt && !profiling_enabled();
  if (cfg.loop == 1 && !graph_possible)
    fail(PVI_ERR_PARAMETER, "graph-resident loop needs no checkpoints");
  // auto: the graph for two-vector tests; the periodic span's 8-branch graph
  // costs more to build than it saves over its typical 12-20 sweeps (c/m5/exp1
  // 40.1 ms host vs 41.7 ms graph on a B200), so it runs only on request
  const bool use_graph = graph_possible && (cfg.loop == 1 || (cfg.loop < 0 && hist_cap == 2));
  std::uint64_t graph_sweeps = 0;
  const auto t_loop_start = std::chrono::steady_clock::now();
  auto nvtx_loop = std::make_unique<NvtxRange>("pvi solve loop");
  while (true) {
    if (cfg.fixed_iterations > 0) {
      if (iteration >= cfg.fixed_iterations) {
        converged = true;
        break;
      }
    } else if (iteration >= start_iteration + cfg.max_iterations) {
      break;
    }
    if (use_graph && sweeps > 0 && static_cast<int>(order.size()) == hist_cap) {
      // every remaining sweep in one graph launch (the first sweep ran eagerly:
      // it builds the per-model tables and scratch the captured sweeps reuse;
      // periodic span: the first 7, which fill the ring)
      const int a_slot = order.front(), b_slot = order.back();
      const std::vector<int> base = order;  // ring oldest..newest at entry
      PoolBuf dls(sizeof(LoopState), stream.s);
      LoopState h{};
      h.iteration = iteration;
      h.limit = cfg.fixed_iterations > 0 ? cfg.fixed_iterations : start_iteration + cfg.max_iterations;
      h.first_bad = ~0ull;
      h.epsilon = cfg.epsilon;
      h.test = cfg.fixed_iterations == 0 ? test : -1;
      h.fixed = cfg.fixed_iterations > 0 ? 1 : 0;
      PVI_CUDA(cudaMemcpyAsync(dls.p, &h, sizeof(h), cudaMemcpyHostToDevice, stream.s));
      cudaGraph_t graph = nullptr;
      const auto tr0 = std::chrono::steady_clock::now();
      PVI_CUDA(cudaGraphCreate(&graph, 0));
      cudaGraphConditionalHandle h_while, h_if;
      PVI_CUDA(cudaGraphConditionalHandleCreate(&h_while, graph, 1, cudaGraphCondAssignDefault));
      if (hist_cap == 2)  // an unused handle fails instantiation (ConditionalHandleUnused)
        PVI_CUDA(cudaGraphConditionalHandleCreate(&h_if, graph, 0, cudaGraphCondAssignDefault));
      cudaGraphNodeParams wp = {};
      wp.type = cudaGraphNodeTypeConditional;
      wp.conditional.handle = h_while;
      wp.conditional.type = cudaGraphCondTypeWhile;
      wp.conditional.size = 1;
      cudaGraphNode_t wnode;
      PVI_CUDA(cudaGraphAddNode(&wnode, graph, nullptr, 0, &wp));
      cudaGraph_t body = wp.conditional.phGraph_out[0];
      auto sweep_args = [&](int from, int to) {
        SweepArgs<T> a;
        a.v = ring[from]->as<T>();
        a.vout = ring[to]->as<T>();
        a.lo = 0;
        a.hi = n;
        a.gamma = gamma;
        a.algorithm = algo;
        a.fa.test = h.test;
        a.fa.gamma = gamma;
        a.fa.stats = dstats.as<SweepStats>();
        a.init_stats = false;  // reset by the decision kernel after every sweep
        return a;
      };
      cudaStream_t cs = stream.s;
      if (hist_cap != 2) {
        // body: IF_0 -> IF_1 -> .. -> IF_7; IF_k { sweep base[k-1] -> base[k]
        // with history base[k+1..k+7], decide } -- the host loop's ring
        // rotation, one phase per slot (IF_0 armed at launch)
        std::vector<cudaGraphConditionalHandle> hk(static_cast<std::size_t>(hist_cap));
        for (int k = 0; k < hist_cap; ++k)
          PVI_CUDA(cudaGraphConditionalHandleCreate(&hk[k], graph, k == 0 ? 1 : 0, cudaGraphCondAssignDefault));
        cudaGraphNode_t prev = nullptr;
        for (int k = 0; k < hist_cap; ++k) {
          cudaGraphNodeParams ip = {};
          ip.type = cudaGraphNodeTypeConditional;
          ip.conditional.handle = hk[k];
          ip.conditional.type = cudaGraphCondTypeIf;
          ip.conditional.size = 1;
          cudaGraphNode_t inode;
          PVI_CUDA(cudaGraphAddNode(&inode, body, prev ? &prev : nullptr, prev ? 1 : 0, &ip));
          prev = inode;
          SweepArgs<T> a = sweep_args(base[(k + hist_cap - 1) % hist_cap], base[k]);
          if (h.test == PVI_TEST_PERIODIC_SPAN) {
            a.fa.n_hist = hist_cap - 1;
            for (int j = 0; j < hist_cap - 1; ++j) a.fa.hist[j] = ring[base[(k + 1 + j) % hist_cap]]->p;
          }
          cudaGraph_t tmp = nullptr;
          PVI_CUDA(cudaStreamBeginCaptureToGraph(cs, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                 cudaStreamCaptureModeRelaxed));
          launch_sweep<T>(m, dm, a, scratch, cs);
          k_loop_decide_phase<<<1, 1, 0, cs>>>(dls.as<LoopState>(), dstats.as<SweepStats>(), h_while, hk[k],
                                               hk[(k + 1) % hist_cap]);
          PVI_CUDA(cudaGetLastError());
          PVI_CUDA(cudaStreamEndCapture(cs, &tmp));
        }
      } else {
      // body: sweep b -> a, decide (sets WHILE and IF), IF { sweep a -> b, decide }
      PVI_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      launch_sweep<T>(m, dm, sweep_args(b_slot, a_slot), scratch, cs);
      k_loop_decide<<<1, 1, 0, cs>>>(dls.as<LoopState>(), dstats.as<SweepStats>(), h_while, h_if, 1);
      PVI_CUDA(cudaGetLastError());
      {
        cudaStreamCaptureStatus cst;
        const cudaGraphNode_t* deps = nullptr;
        std::size_t ndeps = 0;
        cudaGraph_t cap = nullptr;
        PVI_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cap, &deps, &ndeps));
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = h_if;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        cudaGraphNode_t inode;
        PVI_CUDA(cudaGraphAddNode(&inode, cap, deps, ndeps, &ip));
        PVI_CUDA(cudaStreamUpdateCaptureDependencies(cs, &inode, 1, cudaStreamSetCaptureDependencies));
        cudaGraph_t tmp = nullptr;
        PVI_CUDA(cudaStreamEndCapture(cs, &tmp));
        cudaGraph_t ibody = ip.conditional.phGraph_out[0];
        PVI_CUDA(cudaStreamBeginCaptureToGraph(cs, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        launch_sweep<T>(m, dm, sweep_args(a_slot, b_slot), scratch, cs);
        k_loop_decide<<<1, 1, 0, cs>>>(dls.as<LoopState>(), dstats.as<SweepStats>(), h_while, h_if, 0);
        PVI_CUDA(cudaGetLastError());
        PVI_CUDA(cudaStreamEndCapture(cs, &tmp));
      }
      }
      cudaGraphExec_t exec = nullptr;
      const auto tr1 = std::chrono::steady_clock::now();
      {
        cudaGraphInstantiateParams ipar = {};
        const cudaError_t ie = cudaGraphInstantiateWithParams(&exec, graph, &ipar);
        if (ie != cudaSuccess) {
          cudaGraphNodeType nt = cudaGraphNodeTypeEmpty;
          if (ipar.errNode_out) cudaGraphNodeGetType(ipar.errNode_out, &nt);
          cudaGetLastError();
          cudaGraphDestroy(graph);
          fail(PVI_ERR_DEVICE, std::string("graph loop instantiate: ") + cudaGetErrorString(ie) + " (result " +
                                 std::to_string(static_cast<int>(ipar.result_out)) + ", node type " +
                                 std::to_string(static_cast<int>(nt)) + ")");
        }
      }
      const auto tr2 = std::chrono::steady_clock::now();
      PVI_CUDA(cudaEventRecord(ev0, cs));
      init_stats_device(dstats.as<SweepStats>(), cs);  // the first graph sweep's statistics
      PVI_CUDA(cudaGraphLaunch(exec, cs));
      PVI_CUDA(cudaEventRecord(ev1, cs));
      PVI_CUDA(cudaMemcpyAsync(&h, dls.p, sizeof(h), cudaMemcpyDeviceToHost, cs));
      PVI_CUDA(cudaStreamSynchronize(cs));
      const auto tr3 = std::chrono::steady_clock::now();
      cudaGraphExecDestroy(exec);
      cudaGraphDestroy(graph);
      if (loop_trace())
        std::fprintf(stderr, "[pvi loop] capture %.3f ms, instantiate %.3f ms, launch+sync %.3f ms, destroy %.3f ms\n",
                     std::chrono::duration<double, std::milli>(tr1 - tr0).count(),
                     std::chrono::duration<double, std::milli>(tr2 - tr1).count(),
                     std::chrono::duration<double, std::milli>(tr3 - tr2).count(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr3).count());
      float ms = 0.f;
      PVI_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
      sweep_ms += ms;
      graph_sweeps = h.iteration - iteration;
      sweeps += graph_sweeps;
      iteration = h.iteration;
      if (hist_cap != 2) {  // the ring rotated once per graph sweep
        for (int i = 0; i < hist_cap; ++i) order[i] = base[(graph_sweeps + i) % hist_cap];
      } else if (graph_sweeps % 2 == 1) {  // newest is slot a
        order.clear();
        order.push_back(b_slot);
        order.push_back(a_slot);
      }
      if (h.first_bad != ~0ull)
        fail(PVI_ERR_DIVERGENCE, "non-finite value for state " + std::to_string(h.first_bad) +
                                     " at iteration " + std::to_string(h.bad_iteration), h.bad_iteration);
      if (h.test >= 0) {
        last_hi = h.last_hi;
        last_lo = h.last_lo;
      }
      converged = h.converged != 0;
      break;
    }
    ++iteration;
    const int prev_slot = order.back();
    int next_slot;
    if (static_cast<int>(order.size()) < hist_cap) {
      next_slot = static_cast<int>(order.size());
    } else {
      next_slot = order.front();
      order.erase(order.begin());
    }
    const int hist_after = static_cast<int>(order.size()) + 1;
    const bool want_test = cfg.fixed_iterations == 0 && hist_after >= hist_cap;

    SweepArgs<T> a;
    a.v = ring[prev_slot]->as<T>();
    a.vout = ring[next_slot]->as<T>();
    a.lo = 0;
    a.hi = n;
    a.gamma = gamma;
    a.algorithm = algo;
    a.fa.test = want_test ? test : -1;
    a.fa.gamma = gamma;
    a.fa.stats = dstats.as<SweepStats>();
    if (want_test && test == PVI_TEST_PERIODIC_SPAN) {
      // previous vectors oldest..newest, excluding the slot being written
      a.fa.n_hist = static_cast<int>(order.size());
      for (int k = 0; k < a.fa.n_hist; ++k) a.fa.hist[k] = ring[order[k]]->p;
    }
    PVI_CUDA(cudaEventRecord(ev0, stream.s));
    launch_sweep<T>(m, dm, a, scratch, stream.s);
    PVI_CUDA(cudaEventRecord(ev1, stream.s));
    PVI_CUDA(cudaMemcpyAsync(pstats.h, dstats.p, sizeof(SweepStats), cudaMemcpyDeviceToHost, stream.s));
    PVI_CUDA(cudaStreamSynchronize(stream.s));
    float ms = 0.f;
    PVI_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    sweep_ms += ms;
    ++sweeps;
    order.push_back(next_slot);

    if (pstats.h->first_bad != ~0ull)
      fail(PVI_ERR_DIVERGENCE, "non-finite value for state " + std::to_string(pstats.h->first_bad) +
                                   " at iteration " + std::to_string(iteration), iteration);
    if (want_test) {
      last_hi = dkey_inv(pstats.h->max_key);
      last_lo = test == PVI_TEST_VALUE_SPAN ? 0.0 : dkey_inv(pstats.h->min_key);
      converged = evaluate_test(test, last_hi, last_lo, cfg.epsilon, iteration);
    }
    if (ckpt && iteration % cfg.checkpoint_every == 0)
      write_checkpoint(ring[order.back()]->as<T>(), iteration);
    if (converged) break;
  }

  nvtx_loop.reset();
  const auto t_loop_end = std::chrono::steady_clock::now();
  NvtxRange nvtx_extraction("pvi policy extraction + read-back");
  // Policy extraction (vi.hpp:267-280): one more argmax sweep.
  const T* vfinal = ring[order.back()]->as<T>();
  // The value read-back overlaps the extraction sweep (which only reads
  // vfinal): widened on the solve stream, copied out on a side stream.
  std::unique_ptr<PoolBuf> wide;
  std::unique_ptr<Stream> side;
  cudaEvent_t ev_wide = nullptr;
  if (out_values) {
    wide = std::make_unique<PoolBuf>(n * sizeof(double), stream.s);
    launch_widen<T>(vfinal, wide->as<double>(), n, stream.s);
    side = std::make_unique<Stream>();
    PVI_CUDA(cudaEventCreateWithFlags(&ev_wide, cudaEventDisableTiming));
    PVI_CUDA(cudaEventRecord(ev_wide, stream.s));
  }
  PoolBuf policy(n * sizeof(std::uint32_t), stream.s);
  {
    SweepArgs<T> a;
    a.v = vfinal;
    a.act = policy.as<std::uint32_t>();
    a.lo = 0;
    a.hi = n;
    a.gamma = gamma;
    a.algorithm = algo;
    PVI_CUDA(cudaEventRecord(ev0, stream.s));
    launch_sweep<T>(m, dm, a, scratch, stream.s);
    PVI_CUDA(cudaEventRecord(ev1, stream.s));
    if (out_values) {
      PVI_CUDA(cudaStreamWaitEvent(side->s, ev_wide, 0));
      BounceCopier::get().copy(out_values, wide->p, n * 8, side->s);
      cudaEventDestroy(ev_wide);
    }
    PVI_CUDA(cudaStreamSynchronize(stream.s));
    float ms = 0.f;
    PVI_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    sweep_ms += ms;
    ++sweeps;
  }
  wide.reset();  // freed on the solve stream, after the side copy completed
  if (writer) writer->finish();  // every checkpoint on disk before returning
  if (out_policy) BounceCopier::get().copy(out_policy, policy.p, n * 4, stream.s);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  if (loop_trace())
    std::fprintf(stderr, "[pvi loop] setup %.3f ms, loop %.3f ms, extraction+copies %.3f ms\n",
                 std::chrono::duration<double, std::milli>(t_loop_start - t_start).count(),
                 std::chrono::duration<double, std::milli>(t_loop_end - t_loop_start).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_loop_end).count());
  if (stats) {
    stats->iterations = iteration;
    stats->converged = converged ? 1 : 0;
    stats->wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    stats->sweep_seconds = sweep_ms * 1e-3;
    stats->sweeps = sweeps;
    stats->span_lo = last_lo;
    stats->span_hi = last_hi;
    stats->terms_per_sweep = m.terms_per_sweep();
    stats->graph_sweeps = graph_sweeps;
    stats->l2_window_bytes = l2_bytes;
    stats->l2_hit_ratio = l2_ratio;
  }
}

}  // namespace

void vi_solve(const Model& m, const pvi_vi_config& cfg, const double* resume_values,
              std::uint64_t resume_iteration, const std::uint8_t* resume_fp, double* out_values,
              std::uint32_t* out_policy, pvi_vi_stats* stats) {
  if (!(cfg.epsilon > 0.0)) fail(PVI_ERR_PARAMETER, "value iteration: epsilon must be > 0");
  if (cfg.precision == 1)
    solve_impl<float>(m, cfg, resume_values, resume_iteration, resume_fp, out_values, out_policy, stats);
  else
    solve_impl<double>(m, cfg, resume_values, resume_iteration, resume_fp, out_values, out_policy, stats);
}

// ---------------------------------------------------------------------------
// Single sweeps with host buffers

namespace {

// PVI_E2E_PAIRS=0: the host-buffer factored B backup uploads V in
// contiguous quarters instead of x_3-pair blocks
bool e2e_pairs() {
  static const bool on = [] {
    const char* e = std::getenv("PVI_E2E_PAIRS");
    return !(e && e[0] == '0');
  }();
  return on;
}

int backup_chunks() {
  static const int v = [] {
    const char* e = std::getenv("PVI_BACKUP_CHUNKS");
    const int c = e ? std::atoi(e) : 4;
    return std::max(1, std::min(c, Workspace::kChunkEvents));
  }();
  return v;
}

template <typename T>
void backup_impl(const Model& m, double gamma, const void* values, std::uint64_t lo,
                 std::uint64_t hi, void* out_values, std::uint32_t* out_actions, void* out_q) {
  NvtxRange nvtx_range("pvi backup (host buffers)");
  const std::uint64_t n = m.space.count;
  if (lo > hi || hi > n) fail(PVI_ERR_PARAMETER, "state range out of bounds");
  const int device = select_device(-1);
  const DevModel& dm = m.device_view(device);
  Workspace& ws = workspace(m, device);
  std::lock_guard<std::mutex> lock(ws.mu);
  cudaStream_t st = ws.stream;
  T* v = ws.io.get<T>(0, n, st);
  const std::uint64_t nr = hi - lo;
  // Factored B (m = 3, radix-16 orders): stage 1 CTA r reads only
  // V[r |x_b| .. (r+1) |x_b|), so the upload of V is split into pieces and
  // each piece's stage-1 CTAs start as soon as it lands.
  const bool b_pipe = m.scenario == PVI_SCENARIO_B && m.algorithm == PVI_ALGO_FACTORED &&
                      m.pb.useful_life == 3 && m.b_nb == 16 && m.b_na <= 16 && !out_q &&
                      (out_values || out_actions) && n >= (std::uint64_t(1) << 22) && backup_chunks() > 1;
  const int n_pieces = b_pipe ? 4 : 1;
  if (!b_pipe) PVI_CUDA(cudaMemcpyAsync(v, values, n * sizeof(T), cudaMemcpyHostToDevice, st));
  T* vo = out_values ? ws.io.get<T>(1, nr, st) : nullptr;
  std::uint32_t* ao = out_actions ? ws.io.get<std::uint32_t>(2, nr, st) : nullptr;
  T* qo = out_q ? ws.io.get<T>(3, nr * m.n_actions, st) : nullptr;
  maybe_poison(vo, nr * sizeof(T), st);  // debug (PVI_POISON=1): unwritten outputs show up
  maybe_poison(ao, nr * sizeof(std::uint32_t), st);
  maybe_poison(qo, nr * m.n_actions * sizeof(T), st);
  SweepArgs<T> a;
  a.v = v;
  a.vout = vo;
  a.act = ao;
  a.qout = qo;
  a.out_off = lo;
  a.gamma = gamma;
  a.algorithm = m.algorithm;
  a.want_values = out_values || out_actions;
  if (b_pipe && lo == 0 && hi == n && std::is_same<T, double>::value && e2e_pairs() &&
      b_sweep_honours_xb_range(m, device) && m.b_na % 2 == 0 && m.b_na / 2 <= 8) {
    // Pipelined by x_3 pairs.  Stage 2 of the states with top A digit
    // x_3 in {2p, 2p+1} reads the W rows r = (o_a, x_3, x_2) of that pair
    // (and the constants' rows of lower x_3, done by earlier pairs); stage 1
    // builds row r from the V slab r, i.e. the states whose two LOW A digits
    // are (x_3, x_2).  So piece p of V is the 2-D block {top digit t,
    // low digits in pair p}: 16 runs of 32 slabs.  Upload piece p (up
    // stream) -> stage 1 rows of pair p -> stage 2 of pair p -> its V' and
    // argmax (one contiguous range) back on the copy stream, while the next
    // piece uploads and the next pair computes: both PCIe directions and the
    // SMs stay busy.
    const int na = m.b_na, pairs = na / 2;
    const std::uint64_t n_xb = static_cast<std::uint64_t>(m.b_nb) * m.b_nb * m.b_nb;
    const std::uint64_t slab_run = 2ull * na * n_xb;                 // states per (t, pair) run
    const std::uint64_t pitch = static_cast<std::uint64_t>(na) * na * n_xb;  // states per top digit
    const std::uint64_t per_pair = 2 * pitch;                         // output states per pair
    // PVI_LOOP_TRACE=1: timestamps of every piece (timing events, trace only)
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t sm) {
      if (!loop_trace()) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, sm);
      tev.push_back(e);
    };
    mark(st);
    // piece 0 goes up in two halves (top digits t < na/2, then the rest) so
    // the first stage-1 rows start after 1/16 of V instead of 1/8
    const int th = na / 2;
    const std::uint64_t n_r = static_cast<std::uint64_t>(na) * na * na;
    for (int p = 0; p < pairs; ++p) {
      const std::uint64_t off = static_cast<std::uint64_t>(p) * slab_run;
      const T* src = static_cast<const T*>(values);
      if (p == 0) {
        PVI_CUDA(cudaMemcpy2DAsync(v + off, pitch * sizeof(T), src + off, pitch * sizeof(T), slab_run * sizeof(T), th,
                                   cudaMemcpyHostToDevice, ws.up));
        PVI_CUDA(cudaEventRecord(ws.ev[16], ws.up));
        const std::uint64_t off2 = off + th * pitch;
        PVI_CUDA(cudaMemcpy2DAsync(v + off2, pitch * sizeof(T), src + off2, pitch * sizeof(T), slab_run * sizeof(T),
                                   na - th, cudaMemcpyHostToDevice, ws.up));
        PVI_CUDA(cudaEventRecord(ws.ev[17], ws.up));
      } else {
        PVI_CUDA(cudaMemcpy2DAsync(v + off, pitch * sizeof(T), src + off, pitch * sizeof(T), slab_run * sizeof(T), na,
                                   cudaMemcpyHostToDevice, ws.up));
        PVI_CUDA(cudaEventRecord(ws.done[Workspace::kChunkEvents / 2 + p], ws.up));
      }
      mark(ws.up);
    }
    // stage 1 pieces in order on `st`; stage 2 of pair p on s2[] once
    // stage 1 of pieces <= p is done (it also reads the constants' rows of
    // lower pairs), so consecutive grids fill each other's tail
    for (int p = 0; p < pairs; ++p) {
      a.stages = 1;
      a.lo = 0;
      a.hi = n;
      a.x3_rows_lo = 2 * p;
      a.x3_rows_hi = 2 * p + 1;
      if (p == 0) {
        // rows r = (o_a = t, ...): the first half of the rows reads the first half-piece
        PVI_CUDA(cudaStreamWaitEvent(st, ws.ev[16], 0));
        a.r_lo = 0;
        a.r_hi = n_r / na * th;
        launch_sweep<T>(m, dm, a, ws.scratch, st);
        PVI_CUDA(cudaStreamWaitEvent(st, ws.ev[17], 0));
        a.r_lo = a.r_hi;
        a.r_hi = ~0ull;
      } else {
        PVI_CUDA(cudaStreamWaitEvent(st, ws.done[Workspace::kChunkEvents / 2 + p], 0));
      }
      launch_sweep<T>(m, dm, a, ws.scratch, st);
      a.r_lo = 0;
      a.r_hi = ~0ull;
      PVI_CUDA(cudaEventRecord(ws.ev[p], st));
      mark(st);
    }
    // stage 2 of each pair in two x_b column halves: each half's V' / argmax
    // (512 rows of 2,048 states) goes back with one 2-D copy as it finishes
    const std::uint64_t xa_rows = 2ull * na * na;
    for (int p = 0; p < pairs; ++p) {
      // the last pair in quarters: the copy-back that trails the last grid
      // is a quarter of a pair instead of a half
      const int hs = p == pairs - 1 ? 4 : 2;
      for (int h = 0; h < hs; ++h) {
        cudaStream_t cs = ws.s2[(2 * p + h) % 2];
        PVI_CUDA(cudaStreamWaitEvent(cs, ws.ev[p], 0));
        a.stages = 2;
        a.x3_rows_lo = a.x3_rows_hi = -1;
        a.lo = p * per_pair;
        a.hi = (p + 1) * per_pair;
        a.xb_lo = h * n_xb / hs;
        a.xb_hi = (h + 1) * n_xb / hs;
        launch_sweep<T>(m, dm, a, ws.scratch, cs);
        mark(cs);
        PVI_CUDA(cudaEventRecord(ws.ev[20 + 4 * p + h], cs));
        PVI_CUDA(cudaStreamWaitEvent(ws.copy, ws.ev[20 + 4 * p + h], 0));
        PVI_CUDA(cudaStreamWaitEvent(ws.copy2, ws.ev[20 + 4 * p + h], 0));
        const std::uint64_t o = a.lo + a.xb_lo, w = a.xb_hi - a.xb_lo;
        if (out_values)
          PVI_CUDA(cudaMemcpy2DAsync(static_cast<T*>(out_values) + o, n_xb * sizeof(T), vo + o, n_xb * sizeof(T),
                                     w * sizeof(T), xa_rows, cudaMemcpyDeviceToHost, ws.copy));
        if (out_actions)
          PVI_CUDA(cudaMemcpy2DAsync(out_actions + o, n_xb * 4, ao + o, n_xb * 4, w * 4, xa_rows,
                                     cudaMemcpyDeviceToHost, ws.copy2));
        mark(ws.copy);
      }
    }
    a.xb_lo = 0;
    a.xb_hi = ~0ull;
    PVI_CUDA(cudaStreamSynchronize(st));
    for (auto x : ws.s2) PVI_CUDA(cudaStreamSynchronize(x));
    PVI_CUDA(cudaStreamSynchronize(ws.copy));
    PVI_CUDA(cudaStreamSynchronize(ws.copy2));
    PVI_CUDA(cudaStreamSynchronize(ws.up));
    if (!tev.empty()) {
      // order: t0, up[0..P), s1[0..P), then per pair: s2 done, d2h done
      std::string line = "[pvi e2e] ms:";
      for (std::size_t i = 1; i < tev.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[0], tev[i]);
        line += " " + std::to_string(ms).substr(0, 6);
        cudaEventDestroy(tev[i]);
      }
      cudaEventDestroy(tev[0]);
      std::fprintf(stderr, "%s\n", line.c_str());
    }
    return;
  }
  if (b_pipe) {
    const std::uint64_t n_xb = static_cast<std::uint64_t>(m.b_nb) * m.b_nb * m.b_nb;
    const std::uint64_t n_r = n / n_xb;
    a.lo = lo;
    a.hi = hi;
    a.stages = 1;
    for (int k = 0; k < n_pieces; ++k) {
      const std::uint64_t r_lo = n_r * k / n_pieces, r_hi = n_r * (k + 1) / n_pieces;
      const std::uint64_t s_lo = r_lo * n_xb, s_hi = r_hi * n_xb;
      PVI_CUDA(cudaMemcpyAsync(v + s_lo, static_cast<const T*>(values) + s_lo, (s_hi - s_lo) * sizeof(T),
                               cudaMemcpyHostToDevice, ws.copy));
      PVI_CUDA(cudaEventRecord(ws.done[Workspace::kChunkEvents / 2 + k], ws.copy));
      PVI_CUDA(cudaStreamWaitEvent(st, ws.done[Workspace::kChunkEvents / 2 + k], 0));
      a.r_lo = r_lo;
      a.r_hi = r_hi;
      launch_sweep<T>(m, dm, a, ws.scratch, st);
    }
    a.stages = 2;
    a.r_lo = 0;
    a.r_hi = ~0ull;
    if (lo == 0 && hi == n && b_sweep_honours_xb_range(m, device)) {
      // stage 2 by x_b column blocks: every block carries the same mix of
      // light and heavy x_3 pairs (a state-range split would not), and a
      // finished block's V' / argmax is a strided column set -- copied back
      // with one 2-D copy while the next block runs
      const std::uint64_t n_xb = static_cast<std::uint64_t>(m.b_nb) * m.b_nb * m.b_nb;
      const std::uint64_t n_xa = n / n_xb;
      const int cols = std::min(backup_chunks(), Workspace::kChunkEvents / 2);
      for (int c = 0; c < cols; ++c) {
        const std::uint64_t x0 = n_xb * c / cols, x1 = n_xb * (c + 1) / cols;
        a.lo = lo;
        a.hi = hi;
        a.xb_lo = x0;
        a.xb_hi = x1;
        launch_sweep<T>(m, dm, a, ws.scratch, st);
        PVI_CUDA(cudaEventRecord(ws.done[c], st));
        PVI_CUDA(cudaStreamWaitEvent(ws.copy, ws.done[c], 0));
        if (out_values)
          PVI_CUDA(cudaMemcpy2DAsync(static_cast<T*>(out_values) + x0, n_xb * sizeof(T), vo + x0,
                                     n_xb * sizeof(T), (x1 - x0) * sizeof(T), n_xa,
                                     cudaMemcpyDeviceToHost, ws.copy));
        if (out_actions)
          PVI_CUDA(cudaMemcpy2DAsync(out_actions + x0, n_xb * 4, ao + x0, n_xb * 4, (x1 - x0) * 4, n_xa,
                                     cudaMemcpyDeviceToHost, ws.copy));
      }
      PVI_CUDA(cudaStreamSynchronize(st));
      PVI_CUDA(cudaStreamSynchronize(ws.copy));
      return;
    }
  }
  // Large sweeps run as a few state-range chunks so the device-to-host copy
  // of a finished chunk's V' / argmax overlaps the next chunk's sweep (the
  // upload of V cannot overlap: every state may read any V entry).  Only for
  // kernels whose cost scales with the range (not the factored C sweep,
  // which builds whole-space tables per launch).
  const std::uint64_t align = m.chunk_align();
  int chunks = 1;
  if (!out_q && (out_values || out_actions) && align > 0 && nr >= 4 * align &&
      nr >= (std::uint64_t(1) << 22))
    chunks = static_cast<int>(std::min<std::uint64_t>(std::min(backup_chunks(), Workspace::kChunkEvents / 2),
                                                      nr / align));
  std::uint64_t c_lo = lo;
  for (int c = 0; c < chunks; ++c) {
    std::uint64_t c_hi = c + 1 == chunks ? hi : lo + nr * (c + 1) / chunks;
    if (c + 1 < chunks) c_hi = std::max(c_lo, c_hi / align * align);
    if (c_hi <= c_lo) continue;
    a.lo = c_lo;
    a.hi = c_hi;
    launch_sweep<T>(m, dm, a, ws.scratch, st);
    if (chunks > 1) {
      PVI_CUDA(cudaEventRecord(ws.done[c], st));
      PVI_CUDA(cudaStreamWaitEvent(ws.copy, ws.done[c], 0));
      const std::uint64_t off = c_lo - lo, len = c_hi - c_lo;
      if (out_values)
        PVI_CUDA(cudaMemcpyAsync(static_cast<T*>(out_values) + off, vo + off, len * sizeof(T),
                                 cudaMemcpyDeviceToHost, ws.copy));
      if (out_actions)
        PVI_CUDA(cudaMemcpyAsync(out_actions + off, ao + off, len * 4, cudaMemcpyDeviceToHost, ws.copy));
    }
    c_lo = c_hi;
  }
  if (chunks == 1) {  // pageable caller buffers go through the pinned ring
    if (out_values) BounceCopier::get().copy(out_values, vo, nr * sizeof(T), st);
    if (out_actions) BounceCopier::get().copy(out_actions, ao, nr * 4, st);
    if (out_q) BounceCopier::get().copy(out_q, qo, nr * m.n_actions * sizeof(T), st);
  }
  PVI_CUDA(cudaStreamSynchronize(st));
  PVI_CUDA(cudaStreamSynchronize(ws.copy));
}

}  // namespace

void vi_backup(const Model& m, int precision, double gamma, const void* values, std::uint64_t lo,
               std::uint64_t hi, void* out_values, std::uint32_t* out_actions, void* out_q) {
  if (precision == 1)
    backup_impl<float>(m, gamma, values, lo, hi, out_values, out_actions, out_q);
  else
    backup_impl<double>(m, gamma, values, lo, hi, out_values, out_actions, out_q);
}

// ---------------------------------------------------------------------------
// check_convergence over explicit host history (vi.hpp:107-158)

namespace {
template <typename T>
bool check_impl(const Model& m, int test, const void* const* history, int n_hist, double gamma,
                double epsilon, std::uint64_t iteration) {
  const int need = test == PVI_TEST_PERIODIC_SPAN ? 8 : 2;
  if (n_hist < need)
    fail(PVI_ERR_CONTRACT, "convergence test needs " + std::to_string(need) +
                               " value vectors, got " + std::to_string(n_hist));
  if (test == PVI_TEST_PERIODIC_SPAN && iteration < 7) return false;
  const std::uint64_t n = m.space.count;
  select_device(-1);
  Stream stream;
  const int used = test == PVI_TEST_PERIODIC_SPAN ? 8 : 2;
  std::vector<std::unique_ptr<DevBuf>> bufs;
  for (int k = 0; k < used; ++k) {
    bufs.push_back(std::make_unique<DevBuf>(n * sizeof(T)));
    PVI_CUDA(cudaMemcpyAsync(bufs.back()->p, history[n_hist - used + k], n * sizeof(T),
                             cudaMemcpyHostToDevice, stream.s));
  }
  DevBuf dstats(sizeof(SweepStats));
  PinnedStats ps;
  FinalizeArgs fa;
  fa.test = test;
  fa.gamma = gamma;
  fa.stats = dstats.as<SweepStats>();
  fa.n_hist = used - 1;
  for (int k = 0; k < used - 1; ++k) fa.hist[k] = bufs[k]->p;
  launch_stats<T>(bufs[used - 1]->as<T>(), bufs[used - 2]->as<T>(), n, fa, stream.s);
  PVI_CUDA(cudaMemcpyAsync(ps.h, dstats.p, sizeof(SweepStats), cudaMemcpyDeviceToHost, stream.s));
  PVI_CUDA(cudaStreamSynchronize(stream.s));
  const double hi = dkey_inv(ps.h->max_key);
  const double lo = test == PVI_TEST_VALUE_SPAN ? 0.0 : dkey_inv(ps.h->min_key);
  return evaluate_test(test, hi, lo, epsilon, iteration);
}
}  // namespace

bool check_convergence(const Model& m, int precision, int test, const void* const* history,
                       int n_hist, double gamma, double epsilon, std::uint64_t iteration) {
  if (precision == 1) return check_impl<float>(m, test, history, n_hist, gamma, epsilon, iteration);
  return check_impl<double>(m, test, history, n_hist, gamma, epsilon, iteration);
}

// ---------------------------------------------------------------------------
// Device-resident sweep of one shard (multi-GPU driver)

namespace {
struct DeviceSweepBufs {
  Scratch scratch;
  std::unique_ptr<DevBuf> st;
  DevBuf* stats() {
    if (!st) st.reset(new DevBuf(sizeof(SweepStats)));
    return st.get();
  }
};
DeviceSweepBufs& device_sweep_bufs(int device) {
  static thread_local std::map<int, DeviceSweepBufs> bufs;
  return bufs[device];
}

__global__ void k_stats_to_doubles(const SweepStats* st, double* out) {
  const SweepStats s = *st;
  out[0] = s.max_key == 0ull ? -1.7976931348623157e308 : dkey_inv(s.max_key);
  out[1] = s.min_key == ~0ull ? -1.7976931348623157e308 : -dkey_inv(s.min_key);
  out[2] = s.first_bad == ~0ull ? -1.7976931348623157e308 : -static_cast<double>(s.first_bad);
  out[3] = 0.0;
}

template <typename T>
void sweep_device_impl(const Model& m, double gamma, const void* vprev, void* vnext,
                       std::uint32_t* act, std::uint64_t lo, std::uint64_t hi, int test,
                       const void* const* hist, int n_hist, int want_stats, double* stats,
                       cudaStream_t stream, const FinalizeArgs* peers = nullptr) {
  int device = 0;
  PVI_CUDA(cudaGetDevice(&device));
  const DevModel& dm = m.device_view(device);
  // per (thread, device) scratch and statistics: the device-resident sweeps
  // of one thread run one at a time per device (they share these buffers;
  // the sharded driver issues them from one thread on one stream)
  DeviceSweepBufs& bufs = device_sweep_bufs(device);
  Scratch& scratch = bufs.scratch;
  DevBuf* dstats = bufs.stats();
  SweepArgs<T> a;
  a.v = static_cast<const T*>(vprev);
  a.vout = static_cast<T*>(vnext);
  a.act = act;
  a.lo = lo;
  a.hi = hi;
  a.out_off = 0;
  a.gamma = gamma;
  a.algorithm = m.algorithm;
  a.want_values = true;
  if (want_stats && stats) {
    a.fa.stats = dstats->as<SweepStats>();
    a.fa.test = test;
    a.fa.gamma = gamma;
    if (test == PVI_TEST_PERIODIC_SPAN) {
      if (n_hist < 7 || !hist) fail(PVI_ERR_CONTRACT, "periodic span needs 7 previous vectors");
      a.fa.n_hist = 7;
      for (int k = 0; k < 7; ++k) a.fa.hist[k] = hist[n_hist - 7 + k];
    }
  }
  if (peers) {
    a.fa.n_peers = peers->n_peers;
    a.fa.peer_all = peers->peer_all;
    for (int q = 0; q < peers->n_peers; ++q) {
      a.fa.peer_v[q] = peers->peer_v[q];
      a.fa.peer_x3_lo[q] = peers->peer_x3_lo[q];
      a.fa.peer_x3_hi[q] = peers->peer_x3_hi[q];
    }
  }
  launch_sweep<T>(m, dm, a, scratch, stream);
  if (want_stats && stats) k_stats_to_doubles<<<1, 1, 0, stream>>>(dstats->as<SweepStats>(), stats);
  PVI_CUDA(cudaGetLastError());
}
}  // namespace

void vi_sweep_device(const Model& m, int precision, double gamma, const void* vprev, void* vnext,
                     std::uint32_t* act, std::uint64_t lo, std::uint64_t hi, int test,
                     const void* const* hist, int n_hist, int want_stats, double* stats,
                     void* stream) {
  if (lo > hi || hi > m.space.count) fail(PVI_ERR_PARAMETER, "state range out of bounds");
  auto st = static_cast<cudaStream_t>(stream);
  if (precision == 1)
    sweep_device_impl<float>(m, gamma, vprev, vnext, act, lo, hi, test, hist, n_hist, want_stats, stats, st);
  else
    sweep_device_impl<double>(m, gamma, vprev, vnext, act, lo, hi, test, hist, n_hist, want_stats, stats, st);
}

// ---------------------------------------------------------------------------
// Unit shards of the factored B x_3-pair sweep.  Unit u = pair * G + g with
// G = |x_b| / 16 column groups: a stage-2 CTA is (pair, x_b), so a shard of
// consecutive units is a few (pair, column-group range) segments, and the
// state space can be cut finer than whole pairs (8 pairs for 8 ranks left
// the heaviest pair 36% above the lightest).

namespace {

struct UnitGeo {
  int na, pairs;
  std::uint64_t n_xb, groups, per_x3, per_pair;
};

UnitGeo unit_geo(const Model& m) {
  if (!b_sweep_honours_xb_range(m, 0))
    fail(PVI_ERR_PARAMETER, "unit shards need the factored Scenario B x_3-pair sweep");
  UnitGeo g;
  g.na = m.b_na;
  g.pairs = (g.na + 1) / 2;
  g.n_xb = static_cast<std::uint64_t>(m.b_nb) * m.b_nb * m.b_nb;
  g.groups = g.n_xb / 16;
  g.per_x3 = static_cast<std::uint64_t>(g.na) * g.na * g.n_xb;
  g.per_pair = 2 * g.per_x3;
  return g;
}

// A unit range as at most three launches' worth of work: a partial pair at
// the head (a column range), a block of whole pairs, a partial pair at the
// tail.  g_lo/g_hi are column groups, p_lo..p_hi pairs (equal for partials).
struct UnitSeg {
  int p_lo, p_hi;
  std::uint32_t g_lo, g_hi;
};

std::vector<UnitSeg> unit_segments(const UnitGeo& g, std::uint64_t u_lo, std::uint64_t u_hi) {
  std::vector<UnitSeg> out;
  const std::uint32_t G = static_cast<std::uint32_t>(g.groups);
  std::uint64_t u = u_lo;
  while (u < u_hi) {
    const int p = static_cast<int>(u / G);
    const std::uint64_t p_start = static_cast<std::uint64_t>(p) * G;
    const std::uint64_t p_end = p_start + G;
    if (u == p_start && u_hi >= p_end) {
      // whole pairs p .. p1 - 1
      const int p1 = static_cast<int>(u_hi / G);
      out.push_back({p, p1 - 1, 0u, G});
      u = static_cast<std::uint64_t>(p1) * G;
    } else {
      const std::uint64_t end = std::min(u_hi, p_end);
      out.push_back({p, p, static_cast<std::uint32_t>(u - p_start), static_cast<std::uint32_t>(end - p_start)});
      u = end;
    }
  }
  return out;
}

void merge_runs(std::vector<std::pair<std::uint64_t, std::uint64_t>>& runs) {
  std::sort(runs.begin(), runs.end());
  std::vector<std::pair<std::uint64_t, std::uint64_t>> out;
  for (const auto& r : runs) {
    if (r.first >= r.second) continue;
    if (!out.empty() && out.back().second >= r.first)
      out.back().second = std::max(out.back().second, r.second);
    else
      out.push_back(r);
  }
  runs.swap(out);
}

// x_3 rows a unit range's stage 1 builds: its pairs' digits, and the
// constants' rows below
std::pair<int, int> unit_x3_range(const UnitGeo& g, std::uint64_t u_lo, std::uint64_t u_hi) {
  const int p0 = static_cast<int>(u_lo / g.groups), p1 = static_cast<int>((u_hi - 1) / g.groups);
  return {2 * p0, std::min(g.na - 1, 2 * p1 + 1)};
}

}  // namespace

std::uint64_t unit_count(const Model& m) {
  const UnitGeo g = unit_geo(m);
  return static_cast<std::uint64_t>(g.pairs) * g.groups;
}

void unit_partition(const Model& m, int parts, std::uint64_t* bounds) {
  if (parts < 1) fail(PVI_ERR_PARAMETER, "partition: parts must be >= 1");
  const UnitGeo g = unit_geo(m);
  const std::uint64_t nu = static_cast<std::uint64_t>(g.pairs) * g.groups;
  // per-unit cost: the pair's stage-2 diagonal work plus its constants,
  // fitted to per-shard stage-2 times on a B200 (8 unit shards: a pair-7
  // CTA costs ~1.15x a pair-0 CTA, not the 1.38x the FMA counts give: the
  // constants' j loop overlaps the row copies)
  std::vector<double> prefix(nu + 1, 0.0);
  for (std::uint64_t u = 0; u < nu; ++u) {
    const int p = static_cast<int>(u / g.groups);
    prefix[u + 1] = prefix[u] + 34.4 + 0.8 * (p + 1);
  }
  bounds[0] = 0;
  for (int k = 1; k < parts; ++k) {
    const double target = prefix[nu] * k / parts;
    const std::uint64_t u = static_cast<std::uint64_t>(
        std::lower_bound(prefix.begin(), prefix.end(), target) - prefix.begin());
    bounds[k] = std::max(bounds[k - 1], std::min(u, nu));
  }
  bounds[parts] = nu;
}

std::vector<std::pair<std::uint64_t, std::uint64_t>> unit_own_runs(const Model& m, std::uint64_t u_lo,
                                                                   std::uint64_t u_hi) {
  const UnitGeo g = unit_geo(m);
  std::vector<std::pair<std::uint64_t, std::uint64_t>> runs;
  for (const UnitSeg& sg : unit_segments(g, u_lo, u_hi)) {
    const std::uint64_t xa0 = static_cast<std::uint64_t>(2 * sg.p_lo) * g.na * g.na;
    const std::uint64_t xa1 = std::min<std::uint64_t>(static_cast<std::uint64_t>(2 * sg.p_hi + 2) * g.na * g.na,
                                                      static_cast<std::uint64_t>(g.na) * g.na * g.na);
    for (std::uint64_t xa = xa0; xa < xa1; ++xa)
      runs.emplace_back(xa * g.n_xb + 16ull * sg.g_lo, xa * g.n_xb + 16ull * sg.g_hi);
  }
  merge_runs(runs);
  return runs;
}

std::vector<std::pair<std::uint64_t, std::uint64_t>> unit_read_runs(const Model& m, std::uint64_t u_lo,
                                                                    std::uint64_t u_hi) {
  const UnitGeo g = unit_geo(m);
  auto runs = unit_own_runs(m, u_lo, u_hi);
  if (u_lo >= u_hi) return runs;
  const auto x3 = unit_x3_range(g, u_lo, u_hi);
  const int n_r = g.na * g.na * g.na;
  for (int r = 0; r < n_r; ++r) {
    const int ap = r % (g.na * g.na), x2r = ap % g.na, x3r = ap / g.na;
    if ((x3r >= x3.first && x3r <= x3.second) || (x2r == 0 && x3r <= x3.second))
      runs.emplace_back(static_cast<std::uint64_t>(r) * g.n_xb, static_cast<std::uint64_t>(r + 1) * g.n_xb);
  }
  merge_runs(runs);
  return runs;
}

namespace {

template <typename T>
void sweep_units_impl(const Model& m, double gamma, const void* vprev, void* vnext, std::uint32_t* act,
                      std::uint64_t u_lo, std::uint64_t u_hi, int test, int want_stats, double* stats,
                      cudaStream_t stream, const FinalizeArgs& peers) {
  const UnitGeo g = unit_geo(m);
  int device = 0;
  PVI_CUDA(cudaGetDevice(&device));
  const DevModel& dm = m.device_view(device);
  // per (thread, device) scratch and statistics: the device-resident sweeps
  // of one thread run one at a time per device (they share these buffers;
  // the sharded driver issues them from one thread on one stream)
  DeviceSweepBufs& bufs = device_sweep_bufs(device);
  Scratch& scratch = bufs.scratch;
  DevBuf* dstats = bufs.stats();
  const std::uint64_t n = m.space.count;
  bool first = true;
  const bool st_on = want_stats && stats;
  if (st_on && test == PVI_TEST_PERIODIC_SPAN) fail(PVI_ERR_PARAMETER, "unit sweep: periodic span not supported");
  if (st_on) {
    // the reduction of an empty range still has to publish its identity
    init_stats_device(dstats->as<SweepStats>(), stream);
    first = false;
  }
  const auto segs = unit_segments(g, u_lo, u_hi);
  if (!segs.empty()) {
    const UnitSeg& s0 = segs.front();
    const UnitSeg& s1 = segs.back();
    const std::uint32_t G = static_cast<std::uint32_t>(g.groups);
    // stage 1: every row of the shard's pairs and the constants' rows below,
    // in one launch; the non-constant rows of a partial head / tail pair
    // only for its columns
    SweepArgs<T> a;
    a.v = static_cast<const T*>(vprev);
    a.vout = static_cast<T*>(vnext);
    a.out_off = 0;
    a.gamma = gamma;
    a.algorithm = PVI_ALGO_FACTORED;
    a.want_values = true;
    a.stages = 1;
    a.lo = 0;
    a.hi = n;
    a.x3_rows_lo = 2 * s0.p_lo;
    a.x3_rows_hi = std::min(g.na - 1, 2 * s1.p_hi + 1);
    a.x3_rows_strict = 0;
    if (s0.g_lo > 0 || (s0.p_lo == s1.p_hi && s0.g_hi < G)) {
      a.head_pair = s0.p_lo;
      a.head_g_lo = static_cast<int>(s0.g_lo);
    }
    if (s1.g_hi < G) {
      a.tail_pair = s1.p_hi;
      a.tail_g_hi = static_cast<int>(s1.g_hi);
    }
    launch_sweep<T>(m, dm, a, scratch, stream);
    // stage 2: one 1-D grid over the shard's (pair, x_b) units, fused
    // finalize (+ peer stores)
    SweepArgs<T> b;
    b.v = a.v;
    b.vout = a.vout;
    b.act = act;
    b.out_off = 0;
    b.gamma = gamma;
    b.algorithm = PVI_ALGO_FACTORED;
    b.want_values = true;
    b.stages = 2;
    b.lo = 0;
    b.hi = n;
    b.flat_lo = u_lo * 16;
    b.flat_hi = u_hi * 16;
    b.fa = peers;
    if (st_on) {
      b.fa.stats = dstats->as<SweepStats>();
      b.fa.test = test;
      b.fa.gamma = gamma;
    }
    b.init_stats = first;
    launch_sweep<T>(m, dm, b, scratch, stream);
  }
  if (st_on) k_stats_to_doubles<<<1, 1, 0, stream>>>(dstats->as<SweepStats>(), stats);
  PVI_CUDA(cudaGetLastError());
}

}  // namespace

void vi_sweep_device_units(const Model& m, int precision, double gamma, const void* vprev, void* vnext,
                           std::uint32_t* act, std::uint64_t u_lo, std::uint64_t u_hi, int test, int want_stats,
                           double* stats, void* stream, int n_peers, void* const* peer_vnext,
                           const std::uint64_t* peer_u_lo, const std::uint64_t* peer_u_hi) {
  const UnitGeo g = unit_geo(m);
  const std::uint64_t nu = static_cast<std::uint64_t>(g.pairs) * g.groups;
  if (u_lo > u_hi || u_hi > nu) fail(PVI_ERR_PARAMETER, "unit range out of bounds");
  if (n_peers < 0 || n_peers > 8) fail(PVI_ERR_PARAMETER, "between 0 and 8 peers");
  if (precision == 1) fail(PVI_ERR_PARAMETER, "unit shards run the f64 sweep");
  FinalizeArgs pf;
  pf.n_peers = n_peers;
  for (int q = 0; q < n_peers; ++q) {
    if (!peer_vnext[q] || peer_u_lo[q] >= peer_u_hi[q] || peer_u_hi[q] > nu)
      fail(PVI_ERR_PARAMETER, "bad peer descriptor");
    const auto x3 = unit_x3_range(g, peer_u_lo[q], peer_u_hi[q]);
    pf.peer_v[q] = peer_vnext[q];
    pf.peer_x3_lo[q] = x3.first;
    pf.peer_x3_hi[q] = x3.second;
  }
  sweep_units_impl<double>(m, gamma, vprev, vnext, act, u_lo, u_hi, test, want_stats, stats,
                           static_cast<cudaStream_t>(stream), pf);
}

void vi_sweep_device_peers(const Model& m, int precision, double gamma, const void* vprev, void* vnext,
                           std::uint64_t lo, std::uint64_t hi, int test, int want_stats, double* stats,
                           void* stream, int n_peers, void* const* peer_vnext, const std::uint64_t* peer_lo,
                           const std::uint64_t* peer_hi) {
  if (lo > hi || hi > m.space.count) fail(PVI_ERR_PARAMETER, "state range out of bounds");
  if (n_peers < 0 || n_peers > 8) fail(PVI_ERR_PARAMETER, "between 0 and 8 peers");
  if (test == PVI_TEST_PERIODIC_SPAN) fail(PVI_ERR_PARAMETER, "peer sweep: periodic span not supported");
  int device = 0;
  PVI_CUDA(cudaGetDevice(&device));
  FinalizeArgs pf;
  pf.n_peers = n_peers;
  if (!b_sweep_honours_xb_range(m, device)) {
    // every other sweep gathers from all of V: broadcast each finished V'
    // entry of [lo, hi) into every peer's replica
    pf.peer_all = 1;
    for (int q = 0; q < n_peers; ++q) {
      if (!peer_vnext[q] || peer_hi[q] > m.space.count) fail(PVI_ERR_PARAMETER, "bad peer descriptor");
      pf.peer_v[q] = peer_vnext[q];
    }
    auto st = static_cast<cudaStream_t>(stream);
    if (precision == 1)
      sweep_device_impl<float>(m, gamma, vprev, vnext, nullptr, lo, hi, test, nullptr, 0, want_stats, stats, st, &pf);
    else
      sweep_device_impl<double>(m, gamma, vprev, vnext, nullptr, lo, hi, test, nullptr, 0, want_stats, stats, st, &pf);
    return;
  }
  const int na = m.b_na;
  const std::uint64_t n_xb = static_cast<std::uint64_t>(m.b_nb) * m.b_nb * m.b_nb;
  const std::uint64_t per = static_cast<std::uint64_t>(na) * na * n_xb;
  for (int q = 0; q < n_peers; ++q) {
    if (!peer_vnext[q] || peer_lo[q] >= peer_hi[q] || peer_hi[q] > m.space.count)
      fail(PVI_ERR_PARAMETER, "bad peer descriptor");
    pf.peer_v[q] = peer_vnext[q];
    pf.peer_x3_lo[q] = static_cast<int>(peer_lo[q] / per) / 2 * 2;
    pf.peer_x3_hi[q] = std::min(na - 1, static_cast<int>((peer_hi[q] - 1) / per) / 2 * 2 + 1);
  }
  auto st = static_cast<cudaStream_t>(stream);
  if (precision == 1)
    sweep_device_impl<float>(m, gamma, vprev, vnext, nullptr, lo, hi, test, nullptr, 0, want_stats, stats, st, &pf);
  else
    sweep_device_impl<double>(m, gamma, vprev, vnext, nullptr, lo, hi, test, nullptr, 0, want_stats, stats, st, &pf);
}

// ---------------------------------------------------------------------------
// Cost-weighted contiguous partition

void partition(const Model& m, int parts, std::uint64_t* bounds) {
  if (parts < 1) fail(PVI_ERR_PARAMETER, "partition: parts must be >= 1");
  const std::uint64_t n = m.space.count;
  if (c_weekday_local(m)) {
    // factored C: whole weekdays (a shard's tables are its weekdays' rows,
    // launch_c_factored); 7 weekdays over `parts` ranks, sizes differ by <= 1
    const std::uint64_t w = n / 7;
    bounds[0] = 0;
    for (int p = 1; p <= parts; ++p) bounds[p] = std::min<std::uint64_t>(7, (7ull * p + parts - 1) / parts) * w;
    bounds[parts] = n;
    return;
  }
  const std::uint64_t tile = std::max<std::uint64_t>(1, m.tile_states());
  const std::uint64_t n_tiles = (n + tile - 1) / tile;
  std::vector<double> cost(n_tiles, 0.0);
  if (m.scenario == PVI_SCENARIO_B) {
    for (std::uint64_t s = 0; s < n; ++s) cost[s / tile] += m.state_cost(s);
  } else {
    for (std::uint64_t t = 0; t < n_tiles; ++t)
      cost[t] = static_cast<double>(std::min(n, (t + 1) * tile) - t * tile);
  }
  double total = 0.0;
  for (double c : cost) total += c;
  bounds[0] = 0;
  double acc = 0.0;
  std::uint64_t t = 0;
  for (int p = 1; p < parts; ++p) {
    const double target = total * p / parts;
    while (t < n_tiles && acc + cost[t] * 0.5 < target) acc += cost[t++];
    bounds[p] = std::min(n, t * tile);
  }
  bounds[parts] = n;
  for (int p = 1; p <= parts; ++p) bounds[p] = std::max(bounds[p], bounds[p - 1]);
}

}  // namespace pvi_b200
