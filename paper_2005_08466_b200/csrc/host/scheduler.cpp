// Scheduler and the NDRange partitioner.
//
// One rate model drives every decision: rate(device, kernel) is the device's
// EMA-profiled throughput for the kernel (work units per second; alpha = 0.3,
// the first sample sets it -- proj/src/scheduler.cpp:136-149), else its
// modeled rate (relative throughput x baseline). From it:
//   * placement of a whole launch (the reference's four built-in policies,
//     same semantics: user_directed, round_robin, static_map and the
//     residency-aware cost model time = work / rate (+ bytes / bandwidth when
//     the inputs are not resident) with the lowest id winning ties --
//     scheduler.cpp:38-48, 81-106), plus user-registered policies;
//   * partition_weights for a partitioned NDRange: the same rates as integer
//     split weights, so a device twice
//     as fast gets twice the rows.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <limits>
#include <mutex>

#include "haocl/runtime.hpp"
#include "hcl_host.h"

namespace haocl {

const char* error_code_name(ErrorCode code) {
  static const char* names[] = {"internal", "protocol", "version", "malformed", "encoding", "unknown_call",
                                "busy", "precondition", "reassembly_conflict", "argument", "name", "config",
                                "connect", "timeout", "transport", "remote", "handle", "policy", "size",
                                "mapping", "unknown_device", "registration", "contract", "parse"};
  auto i = static_cast<size_t>(code);
  return i < sizeof(names) / sizeof(names[0]) ? names[i] : "unknown";
}

[[noreturn]] static void fail(ErrorCode code, const std::string& m) { throw Error(code, m); }

DeviceState* ClusterState::find(int global_id) {
  for (auto& d : devices)
    if (d.global_id == global_id) return &d;
  return nullptr;
}
const DeviceState* ClusterState::find(int global_id) const {
  for (const auto& d : devices)
    if (d.global_id == global_id) return &d;
  return nullptr;
}

namespace {

// rate(device, kernel): profiled EMA rate, else the device model's rate
double rate_of(const DeviceState& d, const std::string& kernel, const SchedulerOptions& o) {
  auto it = d.profiled_rate.find(kernel);
  return it != d.profiled_rate.end() ? it->second : d.model.relative_throughput * o.baseline_rate;
}

bool inputs_resident_on(const DeviceState& d, const KernelTask& task) {
  return std::all_of(task.args.begin(), task.args.end(),
                     [&](const Arg& a) { return !a.is_buffer || d.resident_buffers.count(a.buffer) > 0; });
}

enum class Builtin { user_directed, round_robin, static_map, cost_model };
constexpr std::pair<const char*, Builtin> kBuiltins[] = {{"user_directed", Builtin::user_directed},
                                                         {"round_robin", Builtin::round_robin},
                                                         {"static_map", Builtin::static_map},
                                                         {"cost_model", Builtin::cost_model}};

const DeviceState& require_device(const ClusterState& st, int gid, const std::string& who) {
  const DeviceState* d = st.find(gid);
  if (!d) fail(ErrorCode::unknown_device, who + ": device " + std::to_string(gid) + " is not in the device map");
  return *d;
}

}  // namespace

struct Scheduler::Impl {
  SchedulerOptions options;
  std::map<std::string, int> kernel_map;     // static_map: kernel -> device
  std::map<std::string, PolicyFn> custom;    // register_policy
  std::atomic<uint64_t> turn{0};             // round_robin
  mutable std::mutex mu;
  ClusterState state;

  static const Builtin* builtin(const std::string& name) {
    for (const auto& [n, b] : kBuiltins)
      if (name == n) return &b;
    return nullptr;
  }

  int place(Builtin b, const KernelTask& task, const TaskEstimate& est) {
    switch (b) {
      case Builtin::user_directed:
        if (task.placement.mode != Placement::Mode::explicit_device)
          fail(ErrorCode::policy, "user_directed placement needs an explicit device id");
        return require_device(state, task.placement.device_id, "user_directed").global_id;
      case Builtin::round_robin:
        return state.devices[turn.fetch_add(1) % state.devices.size()].global_id;
      case Builtin::static_map: {
        auto it = kernel_map.find(task.kernel_name);
        if (it == kernel_map.end())
          fail(ErrorCode::mapping, "static_map: kernel '" + task.kernel_name + "' is not mapped to a device");
        return require_device(state, it->second, "static_map entry for '" + task.kernel_name + "'").global_id;
      }
      case Builtin::cost_model: {
        // device order is ascending id: the first minimum is the lowest id on ties
        const DeviceState* best = nullptr;
        double best_t = std::numeric_limits<double>::infinity();
        for (const auto& d : state.devices) {
          const double t = Scheduler::modeled_cost(d, task.kernel_name, est, options, inputs_resident_on(d, task));
          if (t < best_t) best_t = t, best = &d;
        }
        if (!best) fail(ErrorCode::precondition, "cost_model: no device has a finite cost");
        return best->global_id;
      }
    }
    fail(ErrorCode::internal, "unreachable placement");
  }
};

Scheduler::Scheduler(SchedulerOptions options, std::map<std::string, int> kernel_map) : impl_(new Impl) {
  impl_->options = options;
  impl_->kernel_map = std::move(kernel_map);
}
Scheduler::~Scheduler() = default;

void Scheduler::configure(SchedulerOptions options, std::map<std::string, int> kernel_map) {
  std::lock_guard lock(impl_->mu);
  impl_->options = options;
  impl_->kernel_map = std::move(kernel_map);
  impl_->custom.clear();
  impl_->turn.store(0);
}

const SchedulerOptions& Scheduler::options() const { return impl_->options; }

double Scheduler::modeled_cost(const DeviceState& device, const std::string& kernel_name, const TaskEstimate& est,
                               const SchedulerOptions& options, bool inputs_resident) {
  const double compute = est.work_units / rate_of(device, kernel_name, options);
  const double transfer =
      inputs_resident ? 0.0 : static_cast<double>(est.in_bytes + est.out_bytes) / options.net_bandwidth;
  return compute + transfer;
}

void Scheduler::register_policy(const std::string& name, PolicyFn policy) {
  std::lock_guard lock(impl_->mu);
  if (Impl::builtin(name) || impl_->custom.count(name))
    fail(ErrorCode::registration, "a policy named '" + name + "' exists already");
  impl_->custom.emplace(name, std::move(policy));
}

bool Scheduler::has_policy(const std::string& name) const {
  std::lock_guard lock(impl_->mu);
  return Impl::builtin(name) || impl_->custom.count(name) > 0;
}

int Scheduler::schedule(const KernelTask& task, const TaskEstimate& estimate) {
  std::lock_guard lock(impl_->mu);
  if (impl_->state.devices.empty()) fail(ErrorCode::precondition, "the scheduler knows no devices");
  const std::string name =
      task.placement.mode == Placement::Mode::explicit_device ? "user_directed" : task.placement.policy;
  int chosen;
  if (const Builtin* b = Impl::builtin(name)) {
    chosen = impl_->place(*b, task, estimate);
  } else {
    auto it = impl_->custom.find(name);
    if (it == impl_->custom.end()) fail(ErrorCode::policy, "no placement policy named '" + name + "'");
    chosen = it->second(task, impl_->state, estimate);
  }
  if (!impl_->state.find(chosen))
    fail(ErrorCode::internal, "policy '" + name + "' returned device " + std::to_string(chosen) +
                                  ", which is not in the device map");
  return chosen;
}

void Scheduler::record_profile(int global_id, const std::string& kernel_name, double work_units,
                               double observed_seconds) {
  if (!(observed_seconds > 0.0)) fail(ErrorCode::precondition, "a profile sample needs a positive duration");
  std::lock_guard lock(impl_->mu);
  DeviceState* d = impl_->state.find(global_id);
  if (!d) fail(ErrorCode::unknown_device, "device " + std::to_string(global_id));
  double sample = work_units / observed_seconds;
  auto it = d->profiled_rate.find(kernel_name);
  if (it == d->profiled_rate.end())
    d->profiled_rate[kernel_name] = sample;
  else
    it->second = impl_->options.ema_alpha * sample + (1.0 - impl_->options.ema_alpha) * it->second;
}

// Persisted profiles (§8(f) 2): one "gid<TAB>kernel<TAB>rate" line per
// (device, kernel) EMA rate, %.17g so a round trip is exact.
std::string Scheduler::export_profiles() const {
  std::lock_guard lock(impl_->mu);
  std::string out;
  char buf[64];
  for (const auto& d : impl_->state.devices)
    for (const auto& [kernel, rate] : d.profiled_rate) {
      std::snprintf(buf, sizeof buf, "\t%.17g\n", rate);
      out += std::to_string(d.global_id) + "\t" + kernel + buf;
    }
  return out;
}

size_t Scheduler::import_profiles(const std::string& text) {
  std::lock_guard lock(impl_->mu);
  size_t n = 0, pos = 0;
  while (pos < text.size()) {
    size_t eol = text.find('\n', pos);
    if (eol == std::string::npos) eol = text.size();
    const std::string line = text.substr(pos, eol - pos);
    pos = eol + 1;
    if (line.empty()) continue;
    const size_t t1 = line.find('\t'), t2 = t1 == std::string::npos ? t1 : line.find('\t', t1 + 1);
    if (t2 == std::string::npos) fail(ErrorCode::parse, "profile line needs gid<TAB>kernel<TAB>rate: " + line);
    char* end = nullptr;
    const long gid = std::strtol(line.c_str(), &end, 10);
    const double rate = std::strtod(line.c_str() + t2 + 1, &end);
    if (!(rate > 0.0)) fail(ErrorCode::parse, "profile rate must be > 0: " + line);
    DeviceState* d = impl_->state.find(static_cast<int>(gid));
    if (!d) continue;  // a device this run does not have
    d->profiled_rate[line.substr(t1 + 1, t2 - t1 - 1)] = rate;
    ++n;
  }
  return n;
}

void Scheduler::sync_devices(const std::vector<std::pair<int, DeviceModel>>& devices) {
  std::lock_guard lock(impl_->mu);
  impl_->state.devices.clear();
  for (const auto& [id, model] : devices) {
    DeviceState d;
    d.global_id = id;
    d.model = model;
    impl_->state.devices.push_back(std::move(d));
  }
}

void Scheduler::note_dispatch(int gid) {
  std::lock_guard lock(impl_->mu);
  if (DeviceState* d = impl_->state.find(gid)) d->outstanding_tasks++;
}
void Scheduler::note_complete(int gid) {
  std::lock_guard lock(impl_->mu);
  if (DeviceState* d = impl_->state.find(gid)) d->outstanding_tasks = std::max(0, d->outstanding_tasks - 1);
}
void Scheduler::note_resident(uint64_t buffer_id, const std::vector<int>& ids) {
  std::lock_guard lock(impl_->mu);
  for (auto& d : impl_->state.devices) d.resident_buffers.erase(buffer_id);
  for (int id : ids)
    if (DeviceState* d = impl_->state.find(id)) d->resident_buffers.insert(buffer_id);
}
void Scheduler::drop_resident(uint64_t buffer_id) {
  std::lock_guard lock(impl_->mu);
  for (auto& d : impl_->state.devices) d.resident_buffers.erase(buffer_id);
}
ClusterState Scheduler::snapshot() const {
  std::lock_guard lock(impl_->mu);
  return impl_->state;
}

std::vector<uint64_t> Scheduler::partition_weights(const std::string& kernel_name, const std::vector<int>& gids) const {
  std::lock_guard lock(impl_->mu);
  std::vector<double> rates;
  for (int g : gids) rates.push_back(rate_of(require_device(impl_->state, g, "partition_weights"), kernel_name,
                                             impl_->options));
  const double mx = rates.empty() ? 1.0 : *std::max_element(rates.begin(), rates.end());
  std::vector<uint64_t> w;
  // 20-bit resolution; identical rates give identical weights (block_range)
  for (double r : rates) w.push_back(std::max<uint64_t>(1, static_cast<uint64_t>(std::llround(r / mx * 1048576.0))));
  return w;
}

std::vector<uint64_t> split_ranges(uint64_t total, const std::vector<uint64_t>& weights) {
  if (weights.empty()) fail(ErrorCode::argument, "split_ranges: no parts");
  unsigned __int128 wsum = 0;
  for (uint64_t w : weights) wsum += w;
  if (wsum == 0) fail(ErrorCode::argument, "split_ranges: weights sum to zero");
  std::vector<uint64_t> b(weights.size() + 1, 0);
  unsigned __int128 acc = 0;
  for (size_t i = 0; i < weights.size(); ++i) {
    acc += weights[i];
    b[i + 1] = static_cast<uint64_t>((static_cast<unsigned __int128>(total) * acc) / wsum);
  }
  return b;
}

std::vector<int64_t> spmv_partition_ranges(int64_t rows, const int64_t* row_ptr, int64_t parts,
                                           const std::vector<uint64_t>& weights) {
  if (parts < 1 || parts > rows) fail(ErrorCode::argument, "partition count out of range");
  if (!weights.empty() && static_cast<int64_t>(weights.size()) != parts)
    fail(ErrorCode::argument, "one weight per part");
  unsigned __int128 wsum = 0;
  for (uint64_t w : weights) wsum += w;
  if (!weights.empty() && wsum == 0) fail(ErrorCode::argument, "weights sum to zero");
  int64_t nnz = row_ptr[rows];
  std::vector<int64_t> out(static_cast<size_t>(parts) + 1);
  out[0] = 0;
  int64_t row = 0;
  for (int64_t p = 0; p + 1 < parts; ++p) {
    int64_t target = weights.empty()
                         ? (nnz + parts - 1) / parts
                         : static_cast<int64_t>((static_cast<unsigned __int128>(static_cast<uint64_t>(nnz)) * weights[p] +
                                                 wsum - 1) / wsum);
    int64_t max_end = rows - (parts - 1 - p);
    int64_t want = row_ptr[row] + target;
    // first e in [row+1, max_end] with row_ptr[e] >= want (greedy sweep stop)
    int64_t lo = row + 1, hi = max_end;
    while (lo < hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (row_ptr[mid] >= want) hi = mid; else lo = mid + 1;
    }
    out[p + 1] = lo;
    row = lo;
  }
  out[parts] = rows;
  return out;
}

}  // namespace haocl

// ---------------------------------------------------------------------------
// device-free C entry points (hcl_host.h)

namespace hcl {
void set_last_error(const std::string& m);
}

namespace {

template <typename F>
int host_guarded(F&& f) {
  try {
    f();
    return HCL_OK;
  } catch (const haocl::Error& e) {
    hcl::set_last_error(e.what());
    return HCL_ERR_BASE + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    hcl::set_last_error(std::string("internal: ") + e.what());
    return HCL_ERR_BASE;
  }
}
}  // namespace

struct hcl_scheduler {
  haocl::Scheduler sched;
};

extern "C" {

int hcl_split_ranges(uint64_t total, const uint64_t* weights, int parts, uint64_t* bounds) {
  return host_guarded([&] {
    auto b = haocl::split_ranges(total, std::vector<uint64_t>(weights, weights + parts));
    std::memcpy(bounds, b.data(), b.size() * sizeof(uint64_t));
  });
}

int hcl_spmv_partition_ranges(int64_t rows, const int64_t* row_ptr, int64_t parts, const uint64_t* weights,
                              int64_t* out) {
  return host_guarded([&] {
    std::vector<uint64_t> w;
    if (weights) w.assign(weights, weights + parts);
    auto r = haocl::spmv_partition_ranges(rows, row_ptr, parts, w);
    std::memcpy(out, r.data(), r.size() * sizeof(int64_t));
  });
}

int hcl_sched_create(const hcl_scheduler_options* opts, const int* gids, const double* rel_tp, int n,
                     const char* const* map_kernels, const int* map_gids, int nmap, hcl_scheduler** out) {
  return host_guarded([&] {
    haocl::SchedulerOptions o;
    if (opts) {
      o.baseline_rate = opts->baseline_rate;
      o.net_bandwidth = opts->net_bandwidth;
      o.ema_alpha = opts->ema_alpha;
    }
    std::map<std::string, int> km;
    for (int i = 0; i < nmap; ++i) km[map_kernels[i]] = map_gids[i];
    auto* s = new hcl_scheduler{haocl::Scheduler(o, km)};
    std::vector<std::pair<int, haocl::DeviceModel>> devs;
    for (int i = 0; i < n; ++i) devs.push_back({gids[i], haocl::DeviceModel{haocl::DeviceType::gpu, rel_tp[i]}});
    s->sched.sync_devices(devs);
    *out = s;
  });
}

int hcl_sched_destroy(hcl_scheduler* s) {
  delete s;
  return HCL_OK;
}

int hcl_sched_schedule(hcl_scheduler* s, const char* kernel, const char* policy, int explicit_device,
                       double work_units, uint64_t in_bytes, uint64_t out_bytes, const uint64_t* buffers,
                       int nbuffers, int* chosen) {
  return host_guarded([&] {
    haocl::KernelTask t;
    t.kernel_name = kernel;
    for (int i = 0; i < nbuffers; ++i) t.args.push_back(haocl::Arg::of_handle(buffers[i]));
    t.placement = (policy && *policy) ? haocl::Placement::auto_with(policy) : haocl::Placement::explicit_on(explicit_device);
    *chosen = s->sched.schedule(t, haocl::TaskEstimate{work_units, in_bytes, out_bytes});
  });
}

int hcl_sched_record_profile(hcl_scheduler* s, int gid, const char* kernel, double work, double seconds) {
  return host_guarded([&] { s->sched.record_profile(gid, kernel, work, seconds); });
}

namespace {
void save_text(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw haocl::Error(haocl::ErrorCode::argument, "cannot write " + path);
  f << text;
}
std::string load_text(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw haocl::Error(haocl::ErrorCode::argument, "cannot read " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}
}  // namespace

int hcl_sched_save_profiles(hcl_scheduler* s, const char* path) {
  return host_guarded([&] { save_text(path, s->sched.export_profiles()); });
}
int hcl_sched_load_profiles(hcl_scheduler* s, const char* path, int* loaded) {
  return host_guarded([&] {
    size_t n = s->sched.import_profiles(load_text(path));
    if (loaded) *loaded = static_cast<int>(n);
  });
}

int hcl_sched_rate(hcl_scheduler* s, int gid, const char* kernel, double* rate) {
  return host_guarded([&] {
    auto st = s->sched.snapshot();
    const auto* d = st.find(gid);
    if (!d) throw haocl::Error(haocl::ErrorCode::unknown_device, "device " + std::to_string(gid));
    auto it = d->profiled_rate.find(kernel);
    *rate = it == d->profiled_rate.end() ? 0.0 : it->second;
  });
}

int hcl_sched_note_resident(hcl_scheduler* s, uint64_t buffer, const int* gids, int n) {
  return host_guarded([&] { s->sched.note_resident(buffer, std::vector<int>(gids, gids + n)); });
}

int hcl_sched_register_fixed_policy(hcl_scheduler* s, const char* name, int gid) {
  return host_guarded([&] {
    s->sched.register_policy(name, [gid](const haocl::KernelTask&, const haocl::ClusterState&,
                                         const haocl::TaskEstimate&) { return gid; });
  });
}

int hcl_sched_modeled_cost(hcl_scheduler* s, int gid, const char* kernel, double work, uint64_t in_bytes,
                           uint64_t out_bytes, int resident, double* cost) {
  return host_guarded([&] {
    auto st = s->sched.snapshot();
    const auto* d = st.find(gid);
    if (!d) throw haocl::Error(haocl::ErrorCode::unknown_device, "device " + std::to_string(gid));
    *cost = haocl::Scheduler::modeled_cost(*d, kernel, haocl::TaskEstimate{work, in_bytes, out_bytes},
                                           s->sched.options(), resident != 0);
  });
}

int hcl_sched_partition_weights(hcl_scheduler* s, const char* kernel, const int* gids, int n, uint64_t* weights) {
  return host_guarded([&] {
    auto w = s->sched.partition_weights(kernel, std::vector<int>(gids, gids + n));
    std::memcpy(weights, w.data(), w.size() * sizeof(uint64_t));
  });
}

}  // extern "C"
