// runtime.cpp -- Context / Function / Operator (host C++).
#include "runtime.hpp"
#include "solver.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "common.hpp"
#include "exchange.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {
std::atomic<i64> g_launches{0};

// NVTX range over one phase of an apply (element kernels / interface sum /
// exchange) for nsys / ncu timelines; header-only NVTX v3, no cost without a tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}
void count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
i64 launch_count() { return g_launches.load(); }

// ---------------------------------------------------------------- buffers
template <typename T>
void DeviceBuffer<T>::reset(std::size_t count) {
  release();
  if (count == 0) return;
  TETMF_CUDA(cudaMalloc(&p_, count * sizeof(T)));
  n_ = count;
}
template <typename T>
void DeviceBuffer<T>::release() {
  if (p_) cudaFree(p_);
  p_ = nullptr;
  n_ = 0;
}
template <typename T>
void DeviceBuffer<T>::upload(const T* host, std::size_t count, cudaStream_t s) {
  reset(count);
  if (count) {
    TETMF_CUDA(cudaMemcpyAsync(p_, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
    TETMF_CUDA(cudaStreamSynchronize(s));
  }
}
template class DeviceBuffer<double>;
template class DeviceBuffer<i64>;
template class DeviceBuffer<unsigned>;
template class DeviceBuffer<MacroDesc>;
template class DeviceBuffer<P1DeviceTable>;
template class DeviceBuffer<N1DeviceTable>;
template class DeviceBuffer<N1GramTable>;
template class DeviceBuffer<P2VTable>;

// ---------------------------------------------------------------- forms
const FormInfo& form_info(Form f) {
  // the reference's kForms (forms.cpp:10-14) plus config 2's P1 -div(k grad)
  static const FormInfo kInfo[4] = {
      {Form::P1Diffusion, "P1", Space::P1, {}},
      {Form::P2VDiffusion, "P2V", Space::P2, {Space::P2}},
      {Form::N1CurlCurlMass, "N1", Space::ND1, {Space::P1, Space::P1}},
      {Form::P1KDiffusion, "P1K", Space::P1, {Space::P1}},
  };
  const int i = static_cast<int>(f);
  if (i < 0 || i > 3) fail_arg("unknown form id " + std::to_string(i));
  return kInfo[i];
}

std::vector<int> partition_macros(int num_macros, int rank, int nranks) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail_arg("partition: bad rank / world size");
  std::vector<int> out;
  const long long b = static_cast<long long>(num_macros) * rank / nranks;
  const long long e = static_cast<long long>(num_macros) * (rank + 1) / nranks;
  for (long long m = b; m < e; ++m) out.push_back(static_cast<int>(m));
  return out;
}

// ---------------------------------------------------------------- context
Context::Context(const std::string& mesh_desc, int device, int rank, int nranks, std::vector<int> macros,
                 int partition)
    : Context(mesh_by_name(mesh_desc), device, rank, nranks, std::move(macros), partition) {}

Context::Context(MacroMesh mesh, int device, int rank, int nranks, std::vector<int> macros, int partition)
    : mesh_((mesh.validate(), std::move(mesh))), topo_(mesh_), device_(device), rank_(rank), nranks_(nranks),
      partition_(partition) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail_arg("context: bad rank / world size");
  if (partition != kPartitionMacro && partition != kPartitionSlab) fail_arg("context: unknown partition");
  if (partition == kPartitionSlab) macros.clear();  // slab partition: every rank stores every macro
  macros_ = macros.empty() && (nranks == 1 || partition == kPartitionSlab) ? partition_macros(mesh_.num_tets(), 0, 1)
                                                                           : std::move(macros);
  std::sort(macros_.begin(), macros_.end());
  for (int m : macros_)
    if (m < 0 || m >= mesh_.num_tets()) fail_arg("context: macro id out of range");
  group_ = geometry_groups(mesh_, macros_, &ngroups_);
  if (device_ >= 0) {
    TETMF_CUDA(cudaSetDevice(device_));
    TETMF_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
    stream_ = own_stream_;
  }
}

Context::~Context() {
  levels_.clear();
  if (switch_event_) cudaEventDestroy(switch_event_);
  if (own_stream_) cudaStreamDestroy(own_stream_);
}

void Context::set_stream(cudaStream_t s) {
  if (device_ < 0) fail_arg("set_stream: planning-only context has no device");
  const cudaStream_t next = s ? s : own_stream_;
  if (next == stream_) return;
  if (!switch_event_) TETMF_CUDA(cudaEventCreateWithFlags(&switch_event_, cudaEventDisableTiming));
  TETMF_CUDA(cudaEventRecord(switch_event_, stream_));
  TETMF_CUDA(cudaStreamWaitEvent(next, switch_event_, 0));
  stream_ = next;
}

void Context::synchronize() const {
  if (device_ >= 0) TETMF_CUDA(cudaStreamSynchronize(stream_));
}

Context::LevelData& Context::level(Space s, int level) {
  const auto key = std::make_pair(static_cast<int>(s), level);
  auto it = levels_.find(key);
  if (it != levels_.end()) return *it->second;
  if (device_ < 0) fail_arg("context has no device (planning-only context)");
  auto ld = std::make_unique<LevelData>();
  ld->lay = LevelLayout::make(s, level, mesh_.num_tets(), macros_);
  const int n = ld->lay.n;
  std::vector<MacroDesc> descs(macros_.size());
  for (std::size_t li = 0; li < macros_.size(); ++li) {
    const int m = macros_[li];
    const auto& t = mesh_.tets[m];
    MacroDesc& d = descs[li];
    std::memset(&d, 0, sizeof(d));
    d.group = group_[li];
    d.dmask = static_cast<int>(topo_.dirichlet_mask[m]);
    for (int r = 0; r < 3; ++r) {
      d.V0[r] = static_cast<i64>(n) * topo_.int_vertices[t[0]][r];
      d.X0[r] = mesh_.vertices[t[0]][r];
      for (int c = 0; c < 3; ++c) {
        d.E[c][r] = topo_.int_vertices[t[c + 1]][r] - topo_.int_vertices[t[0]][r];
        d.dX[c][r] = mesh_.vertices[t[c + 1]][r] - mesh_.vertices[t[0]][r];
      }
    }
  }
  ld->macros.upload(descs.data(), descs.size(), stream_);
  if (partition_ == kPartitionSlab && s != Space::P1)
    fail_arg("slab partition: P1 functions only (the P1 -Laplace stencil apply, config 4)");
  std::vector<int> rank_of(mesh_.num_tets(), -1);
  if (nranks_ == 1 || partition_ == kPartitionSlab) {
    std::fill(rank_of.begin(), rank_of.end(), 0);
  } else {
    for (int r = 0; r < nranks_; ++r)
      for (int m : partition_macros(mesh_.num_tets(), r, nranks_)) rank_of[m] = r;
    for (int m : macros_)
      if (rank_of[m] != rank_) fail_arg("context: multi-rank contexts use the default partition");
  }
  if (s == Space::P1) {
    // the default K1 kernel's task list (the A/B variants' lists are built on
    // first use, ensure_p1_variant_tasks) and K2's
    std::vector<int> tasks;
    build_stencil6_tasks(static_cast<int>(macros_.size()), n, tasks);
    if (partition_ == kPartitionSlab) {
      // keep the boxes of this rank's planes (box heights divide the cuts)
      const auto units = slab_partition(mesh_.num_tets(), n, nranks_);
      std::vector<int> zr(2 * macros_.size(), 0), kept;
      for (const SlabUnit& u : units[rank_]) {
        zr[2 * u.macro] = u.za;
        zr[2 * u.macro + 1] = u.zb;
      }
      for (std::size_t t = 0; t < tasks.size(); t += 4) {
        const int li = tasks[t], z0 = tasks[t + 1];
        if (z0 >= zr[2 * li] && z0 < zr[2 * li + 1]) kept.insert(kept.end(), tasks.begin() + t, tasks.begin() + t + 4);
      }
      tasks.swap(kept);
      ld->zrange.upload(zr.data(), zr.size(), stream_);
    }
    ld->ntasks6 = static_cast<int>(tasks.size() / 4);
    ld->tasks6.upload(tasks.data(), tasks.size(), stream_);
    build_p1k_tasks(static_cast<int>(macros_.size()), n, tasks);
    ld->np1k_tasks = static_cast<int>(tasks.size() / 4);
    ld->p1k_tasks.upload(tasks.data(), tasks.size(), stream_);
    build_p1k_walk_tasks(static_cast<int>(macros_.size()), n, tasks);
    ld->np1k_walk = static_cast<int>(tasks.size() / 4);
    ld->p1k_walk.upload(tasks.data(), tasks.size(), stream_);
    {
      int sms = 148;
      TETMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
      // from the mesh's macro count, not this rank's share: the task size sets
      // the summation order, and a partitioned apply stays bitwise equal to
      // the single-rank one
      ld->p1k_chunk = p1k_cube_chunk(mesh_.num_tets(), n, sms);
    }
    build_p1k_cube_tasks(static_cast<int>(macros_.size()), n, tasks, ld->p1k_chunk);
    ld->np1k_cube = static_cast<int>(tasks.size() / 4);
    ld->p1k_cube.upload(tasks.data(), tasks.size(), stream_);
  } else if (s == Space::ND1) {
    std::vector<int> all, part;
    {
      int sms = 148;
      TETMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
      std::vector<int> locals(macros_.size());
      for (std::size_t li = 0; li < macros_.size(); ++li) locals[li] = static_cast<int>(li);
      ld->fold_chunk = n1_fold_chunk(locals, n, sms);
    }
    ld->group_tasks.assign(ngroups_, {0, 0, 0, 0});
    for (int g = 0; g < ngroups_; ++g) {
      std::vector<int> members;
      for (std::size_t li = 0; li < macros_.size(); ++li)
        if (group_[li] == g) members.push_back(static_cast<int>(li));
      for (int pass = 0; pass < 2; ++pass) {
        build_n1_tasks(members, n, pass, part, ld->fold_chunk);
        ld->group_tasks[g][2 * pass] = static_cast<int>(all.size() / 4);
        ld->group_tasks[g][2 * pass + 1] = static_cast<int>(part.size() / 4);
        all.insert(all.end(), part.begin(), part.end());
      }
    }
    ld->ntasks = static_cast<int>(all.size() / 4);
    ld->tasks.upload(all.data(), all.size(), stream_);
    if (n1_kernel_mode() == 3) {
      std::vector<int> merged;
      for (int pass = 0; pass < 2; ++pass) {
        ld->fold_range[2 * pass] = static_cast<int>(merged.size() / 4);
        ld->fold_group_range.resize(ngroups_, {0, 0, 0, 0});
        for (int g = 0; g < ngroups_; ++g) {
          const auto& gt = ld->group_tasks[g];
          std::vector<int> part(all.begin() + 4 * gt[2 * pass], all.begin() + 4 * (gt[2 * pass] + gt[2 * pass + 1]));
          ld->fold_group_range[g][2 * pass] = static_cast<int>(merged.size() / 4);
          ld->fold_group_range[g][2 * pass + 1] = 0;
          if (part.empty()) continue;
          pad_n1_fold_tasks(part);
          merged.insert(merged.end(), part.begin(), part.end());
          ld->fold_group_range[g][2 * pass + 1] = static_cast<int>(part.size() / 4);
        }
        ld->fold_range[2 * pass + 1] = static_cast<int>(merged.size() / 4) - ld->fold_range[2 * pass];
      }
      ld->fold_tasks.upload(merged.data(), merged.size(), stream_);
    }
  } else if (s == Space::P2) {
    // P2V fold walk (k_p2v_fold.cu): per pass, every geometry group's tasks
    // padded to whole CTAs (a CTA stages its group's table)
    int sms = 148;
    TETMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
    std::vector<int> locals(macros_.size()), merged, part;
    for (std::size_t li = 0; li < macros_.size(); ++li) locals[li] = static_cast<int>(li);
    ld->fold_chunk = p2v_fold_chunk(locals, n, sms);
    for (int pass = 0; pass < 2; ++pass) {
      ld->fold_range[2 * pass] = static_cast<int>(merged.size() / 4);
      for (int g = 0; g < ngroups_; ++g) {
        std::vector<int> members;
        for (std::size_t li = 0; li < macros_.size(); ++li)
          if (group_[li] == g) members.push_back(static_cast<int>(li));
        build_p2v_fold_tasks(members, n, pass, part, ld->fold_chunk);
        if (part.empty()) continue;
        pad_p2v_fold_tasks(part);
        merged.insert(merged.end(), part.begin(), part.end());
      }
      ld->fold_range[2 * pass + 1] = static_cast<int>(merged.size() / 4) - ld->fold_range[2 * pass];
    }
    ld->fold_tasks.upload(merged.data(), merged.size(), stream_);
  }
  {
    // solver slot classes (solver.cu): interior = not in a boundary face plane
    // of any macro holding the carrier (fespace.cpp:207-214, 226), owner =
    // lowest sharing macro id
    std::vector<unsigned char> table(16 * macros_.size(), 0);
    for (std::size_t li = 0; li < macros_.size(); ++li) {
      const int m = macros_[li];
      for (unsigned mask = 1; mask < 16; ++mask) {
        const bool interior = !((topo_.dirichlet_mask[m] >> mask) & 1u);
        const auto& sh = topo_.sharers[m][mask];
        const bool owner = sh.empty() || sh.front() == m;
        table[16 * li + mask] = static_cast<unsigned char>((interior ? 1 : 0) | (owner ? 2 : 0));
      }
    }
    ld->slot_table.upload(table.data(), table.size(), stream_);
    ld->dot_scratch.reset(static_cast<std::size_t>(masked_dot_partials() + 2 * (nranks_ + 1)));
  }
  std::vector<std::vector<SlabUnit>> units;
  if (partition_ == kPartitionSlab) units = slab_partition(mesh_.num_tets(), n, nranks_);
  ld->groups = partition_ == kPartitionSlab ? local_groups_slab(mesh_, topo_, ld->lay, units, rank_)
                                            : local_groups_only(mesh_, topo_, ld->lay, rank_of, rank_);
  ld->group_offsets.upload(ld->groups.offsets.data(), ld->groups.offsets.size(), stream_);
  ld->group_copies.upload(ld->groups.copies.data(), ld->groups.copies.size(), stream_);
  if (ld->lay.total() < (i64(1) << 31)) {
    std::vector<unsigned> pairs;
    std::vector<i64> ro{0}, rc;
    const auto& G = ld->groups;
    for (i64 g = 0; g < G.num_groups(); ++g) {
      const i64 b = G.offsets[g], e = G.offsets[g + 1];
      if (e - b == 2) {
        pairs.push_back(static_cast<unsigned>(G.copies[b]));
        pairs.push_back(static_cast<unsigned>(G.copies[b + 1]));
      } else {
        rc.insert(rc.end(), G.copies.begin() + b, G.copies.begin() + e);
        ro.push_back(static_cast<i64>(rc.size()));
      }
    }
    ld->npairs = static_cast<i64>(pairs.size() / 2);
    ld->nrest = static_cast<i64>(ro.size()) - 1;
    ld->group_pairs.upload(pairs.data(), pairs.size(), stream_);
    ld->rest_offsets.upload(ro.data(), ro.size(), stream_);
    ld->rest_copies.upload(rc.data(), rc.size(), stream_);
    ld->packed = true;
  }
  if (nranks_ > 1)
    ld->exchange = std::make_unique<Exchange>(
        partition_ == kPartitionSlab ? build_exchange_plan_slab(mesh_, topo_, ld->lay, units, rank_)
                                     : build_exchange_plan(mesh_, topo_, ld->lay, rank_of, rank_),
        transport_.get(), exchange_put_);
  auto& ref = *ld;
  levels_.emplace(key, std::move(ld));
  return ref;
}

void Context::ensure_p1_variant_tasks(LevelData& ld) {
  if (ld.variant_tasks_built) return;
  const int nm = static_cast<int>(macros_.size()), n = ld.lay.n;
  std::vector<int> tasks;
  build_stencil2_tasks(nm, n, tasks);
  ld.ntasks = static_cast<int>(tasks.size() / 4);
  ld.tasks.upload(tasks.data(), tasks.size(), stream_);
  build_stencil5_tasks(nm, n, tasks);
  ld.ntasks5 = static_cast<int>(tasks.size() / 4);
  ld.tasks5.upload(tasks.data(), tasks.size(), stream_);
  ld.variant_tasks_built = true;
}

Context::LevelData& Context::ref_level(Space s, int level) {
  LevelData& ld = this->level(s, level);
  if (!ld.ref) {
    ld.ref = std::make_unique<RefNumbering>(build_ref_numbering(mesh_, topo_, ld.lay));
    ld.ref_map.upload(ld.ref->map.data(), ld.ref->map.size(), stream_);
    // owned ids are contiguous: the numbering sorts by owner macro first
    // (fespace.cpp:283-295) and ranks hold contiguous macro ranges
    i64 lo = -1, hi = -1;
    for (i64 e : ld.ref->map)
      if (e >= 0 && (e & 1)) {
        const i64 id = e >> 2;
        lo = lo < 0 ? id : std::min(lo, id);
        hi = std::max(hi, id + 1);
      }
    ld.ref_lo = lo < 0 ? 0 : lo;
    ld.ref_hi = lo < 0 ? 0 : hi;
  }
  return ld;
}

// ---------------------------------------------------------------- function
// Every level buffer carries zeroed guard regions of storage_guard(n)
// doubles before and after the macro blocks: the stencil / cube kernels load
// their register windows without bounds predicates (out-of-lattice values
// only ever meet zero weights), so the windows may touch up to one row plus
// one warp width outside the storage.
void Context::LevelData::interface_sum(double* y, cudaStream_t s, bool signed_values) const {
  if (packed)
    launch_interface_sum_packed(y, group_pairs.get(), npairs, rest_offsets.get(), rest_copies.get(), nrest, s,
                                signed_values);
  else
    launch_interface_sum(y, group_offsets.get(), group_copies.get(), groups.num_groups(), s, signed_values);
}

i64 storage_guard(int n) { return round_up(static_cast<i64>(n) + 96, 32); }

double* Function::data(int level) {
  auto it = data_.find(level);
  if (it != data_.end()) return it->second.get() + storage_guard(1 << level);
  auto& ld = ctx_->level(space_, level);
  const i64 g = storage_guard(ld.lay.n);
  DeviceBuffer<double> buf(static_cast<std::size_t>(ld.lay.total() + 2 * g));
  TETMF_CUDA(cudaMemsetAsync(buf.get(), 0, buf.size() * sizeof(double), ctx_->stream()));
  double* p = buf.get() + g;
  data_.emplace(level, std::move(buf));
  return p;
}

const double* Function::data(int level) const {
  auto it = data_.find(level);
  if (it == data_.end()) fail_arg("function has no data at level " + std::to_string(level));
  return it->second.get() + storage_guard(1 << level);
}

i64 Function::size(int level) const { return ctx_->level(space_, level).lay.total(); }

void Function::fill_seeded(int level, std::uint64_t seed, bool dirichlet_zero) {
  if (ctx_->topo().coord_scale == 0) fail_arg("fill_seeded: mesh vertices are not on a dyadic grid");
  auto& ld = ctx_->level(space_, level);
  double* p = data(level);
  if (ld.lay.macros.empty()) return;
  launch_fill_seeded(p, ld.macros.get(), static_cast<int>(ld.lay.macros.size()), ld.lay.macro_stride, ld.lay.n,
                     static_cast<int>(space_), ld.lay.class_stride, seed, dirichlet_zero, ctx_->stream());
}

void Function::fill_coefficient(int level, CoeffSpec spec) {
  if (space_ == Space::ND1) fail_arg("fill_coefficient: coefficient functions live in P1 or P2");
  if (spec.which < 0 || spec.which > 3) fail_arg("fill_coefficient: unknown coefficient");
  auto& ld = ctx_->level(space_, level);
  double* p = data(level);
  if (ld.lay.macros.empty()) return;
  launch_fill_coeff(p, ld.macros.get(), static_cast<int>(ld.lay.macros.size()), ld.lay.macro_stride, ld.lay.n, spec,
                    ctx_->stream(), space_ == Space::P2 ? ld.lay.class_stride : 0);
}

i64 Function::num_ref_dofs(int level) { return ctx_->ref_level(space_, level).ref->num_dofs; }

void Function::import_ref_device(int level, const double* dev_ref) {
  auto& ld = ctx_->ref_level(space_, level);
  launch_import_ref(data(level), ld.ref_map.get(), ld.lay.total(), dev_ref, ctx_->stream());
}

void Function::export_ref_device(int level, double* dev_ref) {
  auto& ld = ctx_->ref_level(space_, level);
  launch_export_ref(data(level), ld.ref_map.get(), ld.lay.total(), dev_ref, ctx_->stream());
}

void Function::owned_ref_range(int level, i64* lo, i64* hi) {
  if (ctx_->partition() == Context::kPartitionSlab)
    fail_arg("owned reference slices: macro partitions only (a slab rank owns scattered ids)");
  auto& ld = ctx_->ref_level(space_, level);
  *lo = ld.ref_lo;
  *hi = ld.ref_hi;
}

void Function::import_ref_owned(int level, const double* host_owned) {
  i64 lo = 0, hi = 0;
  owned_ref_range(level, &lo, &hi);
  auto& ld = ctx_->ref_level(space_, level);
  const cudaStream_t s = ctx_->stream();
  if (ld.ref_io.size() < static_cast<std::size_t>(hi - lo)) ld.ref_io.reset(static_cast<std::size_t>(hi - lo));
  double* p = data(level);
  if (hi > lo)
    TETMF_CUDA(cudaMemcpyAsync(ld.ref_io.get(), host_owned, (hi - lo) * sizeof(double), cudaMemcpyHostToDevice, s));
  if (ld.lay.total() > 0) launch_import_ref_range(p, ld.ref_map.get(), ld.lay.total(), ld.ref_io.get(), lo, hi, s);
  // ghost copies := owner values: rank-local groups, then across ranks
  launch_interface_owner(p, ld.group_offsets.get(), ld.group_copies.get(), ld.groups.num_groups(), s);
  if (ld.exchange) ld.exchange->broadcast_owner(p, s);
  ctx_->synchronize();
}

void Function::export_ref_owned(int level, double* host_owned) {
  i64 lo = 0, hi = 0;
  owned_ref_range(level, &lo, &hi);
  auto& ld = ctx_->ref_level(space_, level);
  const cudaStream_t s = ctx_->stream();
  if (ld.ref_io.size() < static_cast<std::size_t>(hi - lo)) ld.ref_io.reset(static_cast<std::size_t>(hi - lo));
  if (ld.lay.total() > 0)
    launch_export_ref_range(data(level), ld.ref_map.get(), ld.lay.total(), ld.ref_io.get(), lo, hi, s);
  if (hi > lo)
    TETMF_CUDA(cudaMemcpyAsync(host_owned, ld.ref_io.get(), (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx_->synchronize();
}

void Function::import_ref(int level, const double* host_ref) {
  const i64 nd = num_ref_dofs(level);
  DeviceBuffer<double> tmp(static_cast<std::size_t>(nd));
  TETMF_CUDA(cudaMemcpyAsync(tmp.get(), host_ref, nd * sizeof(double), cudaMemcpyHostToDevice, ctx_->stream()));
  import_ref_device(level, tmp.get());
  ctx_->synchronize();
}

void Function::export_ref(int level, double* host_ref) {
  if (ctx_->nranks() > 1) fail_arg("export_ref: single-rank contexts only (gather on the caller side)");
  const i64 nd = num_ref_dofs(level);
  DeviceBuffer<double> tmp(static_cast<std::size_t>(nd));
  export_ref_device(level, tmp.get());
  TETMF_CUDA(cudaMemcpyAsync(host_ref, tmp.get(), nd * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream()));
  ctx_->synchronize();
}

// ---------------------------------------------------------------- operator
Operator::Operator(Context& ctx, Form form, std::vector<const Function*> coeffs)
    : ctx_(&ctx), form_(form), coeffs_(std::move(coeffs)) {
  const FormInfo& fi = form_info(form);
  if (ctx.partition() == Context::kPartitionSlab && form != Form::P1Diffusion)
    fail_arg("slab partition: the P1 -Laplace operator only (config 4)");

  if (coeffs_.size() != fi.coeffSpaces.size())
    fail_arg(std::string("form ") + fi.name + " expects " + std::to_string(fi.coeffSpaces.size()) +
             " coefficient field(s)");
  for (std::size_t c = 0; c < coeffs_.size(); ++c) {
    if (!coeffs_[c]) fail_arg("missing coefficient field");
    if (&coeffs_[c]->ctx() != ctx_) fail_arg("coefficient field belongs to another context");
    if (coeffs_[c]->space() != fi.coeffSpaces[c]) fail_arg("coefficient field has wrong space or level");
  }
}

Operator::LevelTables& Operator::tables(int level) {
  auto it = tables_.find(level);
  if (it != tables_.end()) return *it->second;
  auto lt = std::make_unique<LevelTables>();
  const int ng = ctx_->num_geometry_groups();
  const auto& macros = ctx_->macros();
  const auto& grp = ctx_->geometry_group();
  if (form_ == Form::P2VDiffusion) {
    std::vector<P2VTable> t(ng);
    std::vector<bool> done(ng, false);
    for (std::size_t li = 0; li < macros.size(); ++li)
      if (!done[grp[li]]) {
        t[grp[li]] = p2v_table(ctx_->mesh(), macros[li], level);
        done[grp[li]] = true;
      }
    lt->p2v.upload(t.data(), t.size(), ctx_->stream());
  } else if (form_ == Form::N1CurlCurlMass) {
    std::vector<N1DeviceTable> t(ng);
    std::vector<bool> done(ng, false);
    for (std::size_t li = 0; li < macros.size(); ++li)
      if (!done[grp[li]]) {
        t[grp[li]] = pack_n1(n1_tables(ctx_->mesh(), macros[li], level));
        done[grp[li]] = true;
      }
    lt->n1.upload(t.data(), t.size(), ctx_->stream());
    std::vector<N1GramTable> gt(ng);
    std::fill(done.begin(), done.end(), false);
    for (std::size_t li = 0; li < macros.size(); ++li)
      if (!done[grp[li]]) {
        gt[grp[li]] = n1_gram_table(ctx_->mesh(), macros[li], level);
        done[grp[li]] = true;
      }
    lt->n1g.upload(gt.data(), gt.size(), ctx_->stream());
  } else {
    std::vector<P1DeviceTable> t(ng);
    std::vector<bool> done(ng, false);
    for (std::size_t li = 0; li < macros.size(); ++li)
      if (!done[grp[li]]) {
        t[grp[li]] = pack_p1(p1_tables(ctx_->mesh(), macros[li], level));
        done[grp[li]] = true;
      }
    lt->p1.upload(t.data(), t.size(), ctx_->stream());
  }
  auto& ref = *lt;
  tables_.emplace(level, std::move(lt));
  return ref;
}

void Operator::check(const Function& src, const Function& dst, int level) const {
  const FormInfo& fi = info();
  if (&src.ctx() != ctx_ || &dst.ctx() != ctx_) fail_arg("apply: functions belong to another context");
  if (src.space() != fi.trial || dst.space() != fi.trial || !src.has_level(level))
    fail_arg("apply: field shape mismatch");
  if (&src == &dst) fail_arg("apply: src and dst must be different functions");

  for (const Function* c : coeffs_)
    if (!c->has_level(level)) fail_arg("coefficient field has wrong space or level");
}

// The element kernels form in-macro offsets in 32 bits (row starts, class
// offsets, stencil windows into the guard regions): one check for all of them.
static void check_offsets_32(const LevelLayout& lay) {
  if (lay.macro_stride + 2 * storage_guard(lay.n) >= (i64(1) << 31))
    fail_arg("level " + std::to_string(lay.level) + ": a macro's storage exceeds the kernels' 32-bit offsets");
}

void Operator::kernel_apply(const double* x, double* y, int level) {
  auto& ld = ctx_->level(info().trial, level);
  check_offsets_32(ld.lay);
  const int nm = static_cast<int>(ld.lay.macros.size());
  const cudaStream_t s = ctx_->stream();
  if (nm == 0) {  // a rank without macros still takes part in the exchange
    if (ld.exchange) ld.exchange->run(y, s);
    return;
  }
  auto& t = tables(level);
  cudaEvent_t ev_stop = nullptr;
  if (profiling_) {
    if (events_used_ == events_.size()) {
      cudaEvent_t a, b;
      TETMF_CUDA(cudaEventCreate(&a));
      TETMF_CUDA(cudaEventCreate(&b));
      events_.emplace_back(a, b);
    }
    TETMF_CUDA(cudaEventRecord(events_[events_used_].first, s));
    ev_stop = events_[events_used_].second;
    ++events_used_;
  }
  if (ctx_->partition() == Context::kPartitionSlab && kernel_variant_ != 0)
    fail_arg("slab partition: the default K1 kernel only");
  if ((form_ == Form::P1Diffusion && ((kernel_variant_ >= 2 && kernel_variant_ <= 4) || kernel_variant_ == 7 ||
                                      kernel_variant_ == 8 || kernel_variant_ > 10)) ||
      (form_ == Form::N1CurlCurlMass && kernel_variant_ >= 2) || (form_ == Form::P2VDiffusion && kernel_variant_ >= 3) ||
      (form_ == Form::P1KDiffusion && kernel_variant_ >= 4))
    fail_arg("kernel variant " + std::to_string(kernel_variant_) + " does not exist for this form");
  if (form_ == Form::P1Diffusion && kernel_variant_ >= 2) ctx_->ensure_p1_variant_tasks(ld);
  // put mode: the default K1 kernel stores the exchange's values into the
  // peers' windows itself (Exchange::fused_begin); the rest use the pack kernel
  const bool fused = form_ == Form::P1Diffusion && kernel_variant_ == 0 && ld.exchange && ctx_->exchange_fused() &&
                     ld.exchange->fusable();
  switch (form_) {
    case Form::P1Diffusion:
      if (kernel_variant_ == 1)
        launch_p1_stencil(x, y, ld.macros.get(), nm, ld.lay.macro_stride, ld.lay.n, t.p1.get(), s);
      else if (kernel_variant_ == 6)
        launch_p1_stencil6(x, y, ld.tasks6.get(), ld.ntasks6, ld.lay.macro_stride, ld.lay.n, nm, t.p1.get(),
                           ld.macros.get(), s);
      else if (kernel_variant_ == 5)
        launch_p1_stencil5(x, y, ld.tasks5.get(), ld.ntasks5, ld.lay.macro_stride, ld.lay.n, nm, t.p1.get(),
                           ld.macros.get(), s);
      else if (kernel_variant_ == 10)
        launch_p1_stencil10(x, y, ld.tasks6.get(), ld.ntasks6, ld.lay.macro_stride, ld.lay.n, nm, t.p1.get(),
                            ld.macros.get(), s);
      else if (kernel_variant_ == 9)
        launch_p1_stencil2(x, y, ld.tasks.get(), ld.ntasks, ld.lay.macro_stride, ld.lay.n, t.p1.get(),
                           ld.macros.get(), s);
      else
        launch_p1_stencil6(x, y, ld.tasks6.get(), ld.ntasks6, ld.lay.macro_stride, ld.lay.n, nm, t.p1.get(),
                           ld.macros.get(), s, ld.zrange.get(),
                           fused ? ld.exchange->fused_begin(static_cast<i64>(nm) * ld.lay.macro_stride) : FusedPut{});
      break;
    case Form::P1KDiffusion:
      if (kernel_variant_ == 1)
        launch_p1k_cubes(x, coeffs_[0]->data(level), y, ld.macros.get(), nm, ld.lay.macro_stride, ld.lay.n,
                         t.p1.get(), s);
      else if (kernel_variant_ == 2)  // round-1 default: one 32-point row segment per warp
        launch_p1k_gather(x, coeffs_[0]->data(level), y, ld.p1k_tasks.get(), ld.np1k_tasks, ld.lay.macro_stride,
                          ld.lay.n, t.p1.get(), ld.macros.get(), s);
      else if (kernel_variant_ == 3)  // round-2 first kernel: the gather walked along y
        launch_p1k_walk(x, coeffs_[0]->data(level), y, ld.p1k_walk.get(), ld.np1k_walk, ld.lay.macro_stride,
                        ld.lay.n, t.p1.get(), ld.macros.get(), s);
      else
        launch_p1k_cube(x, coeffs_[0]->data(level), y, ld.p1k_cube.get(), ld.np1k_cube, ld.lay.macro_stride,
                        ld.lay.n, t.p1.get(), ld.macros.get(), s, ld.p1k_chunk);
      break;
    case Form::N1CurlCurlMass: {
      auto& cl = ctx_->level(Space::P1, level);
      if (kernel_variant_ == 1) {
        launch_n1_cubes(x, coeffs_[0]->data(level), coeffs_[1]->data(level), y, ld.macros.get(), nm,
                        ld.lay.macro_stride, ld.lay.class_stride, cl.lay.macro_stride, ld.lay.n, t.n1.get(), s);
      } else {
        const int rule = rule_index();
        for (int pass = 0; pass < 2; ++pass)
          launch_n1_fold(t.n1g.get(), ld.macros.get(), pass, x, coeffs_[0]->data(level), coeffs_[1]->data(level), y,
                         ld.fold_tasks.get() + 4 * ld.fold_range[2 * pass], ld.fold_range[2 * pass + 1],
                         ld.lay.macro_stride, ld.lay.class_stride, cl.lay.macro_stride, ld.lay.n, rule, s, ld.fold_chunk);
      }
      break;
    }
    case Form::P2VDiffusion:
      if (kernel_variant_ == 1 && rule_index() == 0)
        launch_p2v_cubes(x, coeffs_[0]->data(level), y, ld.macros.get(), nm, ld.lay.macro_stride,
                         ld.lay.class_stride, ld.lay.n, t.p2v.get(), s);
      else if (kernel_variant_ == 0 && rule_index() == 0)  // default: fold walk (exact rule)
        for (int pass = 0; pass < 2; ++pass)
          launch_p2v_fold(t.p2v.get(), ld.macros.get(), pass, x, coeffs_[0]->data(level), y,
                          ld.fold_tasks.get() + 4 * ld.fold_range[2 * pass], ld.fold_range[2 * pass + 1],
                          ld.lay.macro_stride, ld.lay.class_stride, ld.lay.n, s, ld.fold_chunk);
      else  // variant 2 (the cube kernel), and the quadrature rules 1-3 (their 10 x 10
            // moment tables: measured as fast in the cube kernel as in the fold walk)
        launch_p2v_cubes2(x, coeffs_[0]->data(level), y, ld.macros.get(), nm, ld.lay.macro_stride,
                          ld.lay.class_stride, ld.lay.n, t.p2v.get(), rule_index(), s);
      break;
    default:
      fail_internal("kernel_apply: unsupported form");
  }
  if (ev_stop) TETMF_CUDA(cudaEventRecord(ev_stop, s));
  {
    NvtxRange r("tetmf interface sum (K4)");
    ld.interface_sum(y, s);
  }
  if (ld.exchange) {
    NvtxRange r("tetmf exchange");
    if (fused)
      ld.exchange->fused_finish(y, s);
    else
      ld.exchange->run(y, s);
  }
}

void Operator::debug_perturb_table(int level, i64 index, double delta) {
  auto& t = tables(level);
  double* base = nullptr;
  std::size_t count = 0;
  if (form_ == Form::N1CurlCurlMass) {  // the fold kernel's Gram table
    base = reinterpret_cast<double*>(t.n1g.get());
    count = t.n1g.size() * sizeof(N1GramTable) / sizeof(double);
  } else if (form_ == Form::P2VDiffusion) {
    base = reinterpret_cast<double*>(t.p2v.get());
    count = t.p2v.size() * sizeof(P2VTable) / sizeof(double);
  } else {
    base = reinterpret_cast<double*>(t.p1.get());
    count = t.p1.size() * sizeof(P1DeviceTable) / sizeof(double);
  }
  if (index < 0 || static_cast<std::size_t>(index) >= count)
    fail_arg("debug_perturb_table: index out of range (" + std::to_string(count) + " table entries)");
  double v = 0.0;
  const cudaStream_t s = ctx_->stream();
  TETMF_CUDA(cudaMemcpyAsync(&v, base + index, sizeof(double), cudaMemcpyDeviceToHost, s));
  TETMF_CUDA(cudaStreamSynchronize(s));
  v += delta;
  TETMF_CUDA(cudaMemcpyAsync(base + index, &v, sizeof(double), cudaMemcpyHostToDevice, s));
  TETMF_CUDA(cudaStreamSynchronize(s));
}

void Operator::set_quadrature(int degree) {
  if (degree < 0 || degree > 6) fail_arg("quadrature: degree must be 0 (exact) or 1..6");
  quad_degree_ = degree;
}

int Operator::rule_index() const {
  int r = 0;
  if (form_ == Form::N1CurlCurlMass && (quad_degree_ == 1 || quad_degree_ == 2)) r = quad_degree_;
  if (form_ == Form::P2VDiffusion && quad_degree_ >= 1 && quad_degree_ <= 3) r = quad_degree_;
  const bool rule_kernel = kernel_variant_ == 0 || (form_ == Form::P2VDiffusion && kernel_variant_ == 2);
  if (r != 0 && (!rule_kernel || (form_ == Form::N1CurlCurlMass && n1_kernel_mode() != 3)))
    fail_arg("quadrature: under-integrating rules run on the default kernels only (and P2V's cube kernel)");
  return r;
}

void Operator::diagonal(Function& d, int level) {
  if (d.space() != info().trial || &d.ctx() != ctx_) fail_arg("diagonal: function not in the operator's trial space");
  for (const Function* c : coeffs_)
    if (!c->has_level(level)) fail_arg("diagonal: coefficient function has no data at this level");
  auto& ld = ctx_->level(info().trial, level);
  check_offsets_32(ld.lay);
  const int nm = static_cast<int>(ld.lay.macros.size());
  double* y = d.data(level);
  const cudaStream_t s = ctx_->stream();
  if (nm > 0) {
    auto& t = tables(level);
    switch (form_) {
      case Form::P1Diffusion:
        launch_p1_diagonal(y, ld.macros.get(), nm, ld.lay.macro_stride, ld.lay.n, t.p1.get(), s);
        break;
      case Form::P1KDiffusion:
        launch_p1k_diagonal(coeffs_[0]->data(level), y, ld.p1k_tasks.get(), ld.np1k_tasks, ld.lay.macro_stride,
                            ld.lay.n, t.p1.get(), ld.macros.get(), s);
        break;
      case Form::N1CurlCurlMass: {
        auto& cl = ctx_->level(Space::P1, level);
        launch_n1_diagonal(y, coeffs_[0]->data(level), coeffs_[1]->data(level), ld.macros.get(), nm,
                           ld.lay.macro_stride, ld.lay.class_stride, cl.lay.macro_stride, ld.lay.n, t.n1g.get(),
                           rule_index(), s);
        break;
      }
      case Form::P2VDiffusion:
        launch_p2v_diagonal(coeffs_[0]->data(level), y, ld.macros.get(), nm, ld.lay.macro_stride,
                            ld.lay.class_stride, ld.lay.n, t.p2v.get(), rule_index(), s);
        break;
      default:
        fail_arg("diagonal: not available for this form");
    }
  }
  ld.interface_sum(y, s, false);
  if (ld.exchange) ld.exchange->run(y, s, false);
}

Operator::~Operator() {
  for (auto& e : events_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
}

void Operator::set_profiling(bool on) {
  if (on && !profiling_) {
    prof_ms_ = 0.0;
    prof_launches_ = 0;
    events_used_ = 0;
  }
  profiling_ = on;
}

void Operator::kernel_stats(double* total_ms, i64* launches) {
  for (std::size_t i = 0; i < events_used_; ++i) {
    TETMF_CUDA(cudaEventSynchronize(events_[i].second));
    float ms = 0.f;
    TETMF_CUDA(cudaEventElapsedTime(&ms, events_[i].first, events_[i].second));
    prof_ms_ += ms;
    ++prof_launches_;
  }
  events_used_ = 0;
  if (total_ms) *total_ms = prof_ms_;
  if (launches) *launches = prof_launches_;
}

double* Operator::ref_scratch(i64 count) {
  if (ref_scratch_.size() < static_cast<std::size_t>(count)) ref_scratch_.reset(static_cast<std::size_t>(count));
  return ref_scratch_.get();
}

void Operator::apply(const Function& src, Function& dst, int level, Update upd) {
  NvtxRange r(info().name);
  check(src, dst, level);
  const double* x = src.data(level);
  if (upd == Update::Replace) {
    kernel_apply(x, dst.data(level), level);
    return;
  }
  const i64 g = storage_guard(1 << level);
  auto it = scratch_.find(level);
  if (it == scratch_.end()) {
    it = scratch_.emplace(level, DeviceBuffer<double>(static_cast<std::size_t>(dst.size(level) + 2 * g))).first;
    TETMF_CUDA(cudaMemsetAsync(it->second.get(), 0, it->second.size() * sizeof(double), ctx_->stream()));
  }
  kernel_apply(x, it->second.get() + g, level);
  launch_axpy(dst.data(level), it->second.get() + g, 1.0, dst.size(level), ctx_->stream());
}

} // namespace tetmf
