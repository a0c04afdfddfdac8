// runtime.hpp -- host C++ operator / function API over the CUDA kernels.
//
// Mirrors the reference's operator API (FormSystem, forms.hpp:41-89) in the
// level-indexed, macro-primitive form the north star asks for:
//
//   Context    mesh + topology + device + rank partition  (FormSystem ctor
//              inputs: MacroMesh, level; forms.cpp:43-56)
//   Function   level-indexed per-macro lattice storage     (FieldVector,
//              fespace.hpp:69-77, but device-resident and per macro)
//   Operator   form + coefficient functions + tables        (FormSystem +
//              StarTables, forms.cpp:33-41, 69-131)
//   Operator::apply(src, dst, level, update)                (FormSystem::apply
//              forms.cpp:195-255: REPLACE; generated kernel_apply ir.cpp:732:
//              ADD)
//
// Errors: std::invalid_argument for wrong space/level/coefficients (as the
// reference), std::logic_error for internal inconsistency, DeviceError /
// CommError for CUDA / NCCL failures. Not thread-safe per object (the
// reference's const methods mutate caches too, forms.hpp:86-87).
#pragma once

#include <array>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "device.hpp"
#include "layout.hpp"
#include "mesh.hpp"
#include "tables.hpp"
#include "common.hpp"
#include "transport.hpp"

namespace tetmf {

template <typename T>
class DeviceBuffer {
public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t count) { reset(count); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) { release(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
    return *this;
  }
  void reset(std::size_t count);
  void release();
  void upload(const T* host, std::size_t count, cudaStream_t s);
  T* get() const { return p_; }
  std::size_t size() const { return n_; }

private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

enum class Form : int { P1Diffusion = 0, P2VDiffusion = 1, N1CurlCurlMass = 2, P1KDiffusion = 3 };
enum class Update : int { Replace = 0, Add = 1 };

struct FormInfo {
  Form id;
  const char* name;
  Space trial;
  std::vector<Space> coeffSpaces;
};
const FormInfo& form_info(Form f);

class Exchange;  // multi-rank interface exchange (exchange.hpp)

class Context {
public:
  // macros: the macro ids this rank stores (empty = all, single rank)
  // partition: kPartitionMacro (whole macros per rank, `macros` = this
  // rank's) or kPartitionSlab ((macro, z-slab) units of P1 points, every
  // rank stores every macro; exchange.hpp slab_partition)
  static constexpr int kPartitionMacro = 0, kPartitionSlab = 1;
  Context(const std::string& mesh_desc, int device, int rank, int nranks, std::vector<int> macros,
          int partition = kPartitionMacro);
  // an in-memory mesh (FormSystem(Form, const MacroMesh&, int), forms.hpp:46);
  // validated like the reference's (mesh.cpp:76-94)
  Context(MacroMesh mesh, int device, int rank, int nranks, std::vector<int> macros,
          int partition = kPartitionMacro);
  int partition() const { return partition_; }
  ~Context();

  const MacroMesh& mesh() const { return mesh_; }
  const Topology& topo() const { return topo_; }
  int device() const { return device_; }
  int rank() const { return rank_; }
  int nranks() const { return nranks_; }
  const std::vector<int>& macros() const { return macros_; }
  const std::vector<int>& geometry_group() const { return group_; }  // per local macro
  int num_geometry_groups() const { return ngroups_; }
  cudaStream_t stream() const { return stream_; }
  // s == nullptr selects the context's own stream (tetmf_ctx_set_stream);
  // work already queued on the old stream is ordered before anything the new
  // stream runs afterwards (event record + stream wait)
  void set_stream(cudaStream_t s);
  void synchronize() const;

  struct LevelData {
    LevelLayout lay;
    DeviceBuffer<MacroDesc> macros;
    InterfaceGroups groups;
    DeviceBuffer<i64> group_offsets, group_copies;
    // K4 fast path: two-copy groups as packed 32-bit (index << 1 | sign)
    // pairs; the groups with more copies keep the CSR form (rest_*). Used
    // when the level's storage has < 2^31 entries, else the full CSR.
    DeviceBuffer<unsigned> group_pairs;
    DeviceBuffer<i64> rest_offsets, rest_copies;
    i64 npairs = 0, nrest = 0;
    bool packed = false;
    void interface_sum(double* y, cudaStream_t s, bool signed_values = true) const;
    std::unique_ptr<RefNumbering> ref;  // lazily, import/export only
    DeviceBuffer<i64> ref_map;
    i64 ref_lo = 0, ref_hi = 0;         // this rank's owned slice of the reference numbering
    DeviceBuffer<double> ref_io;        // staging of the owned slice (host I/O)
    std::unique_ptr<Exchange> exchange; // nranks > 1
    DeviceBuffer<int> tasks;            // kernel task list (per space / level)
    int ntasks = 0;
    DeviceBuffer<int> tasks5;           // P1: interior row-walk CTA tasks (variant 5)
    int ntasks5 = 0;
    DeviceBuffer<int> tasks6;           // P1: shared-memory box tasks (variant 6)
    int ntasks6 = 0;
    bool variant_tasks_built = false;   // P1: the A/B variants' lists (built on first use)
    DeviceBuffer<int> zrange;           // slab partition: per local macro {za, zb} computed here
    DeviceBuffer<int> p1k_tasks;        // P1: row tasks of the P1K gather kernel (K2 round 1, diagonal)
    int np1k_walk = 0;
    DeviceBuffer<int> p1k_walk;         // P1: column-walk tasks of the P1K walk kernel (K2 variant 3)
    int np1k_cube = 0;
    int p1k_chunk = 16;                 // rows = layers per cube-walk task (p1k_cube_chunk)
    DeviceBuffer<int> p1k_cube;         // P1: cube-walk tasks of the P1K cube kernel (K2 default)
    int np1k_tasks = 0;
    // solver (solver.hpp): per local macro, [support mask] -> {bit 0 interior,
    // bit 1 owner copy}; reduction scratch
    DeviceBuffer<unsigned char> slot_table;
    DeviceBuffer<double> dot_scratch;
    // ND1: task ranges (offset, count) per (geometry group, parity pass)
    std::vector<std::array<int, 4>> group_tasks;  // {offset0, count0, offset1, count1}
    // ND1, folded kernel: per pass, all groups' tasks padded to whole CTAs
    DeviceBuffer<int> fold_tasks;
    std::array<int, 4> fold_range{0, 0, 0, 0};    // {offset0, count0, offset1, count1}
    int fold_chunk = 32;                          // steps per fold task (n1_fold_chunk)
    std::vector<std::array<int, 4>> fold_group_range;  // per geometry group, same layout
  };
  LevelData& level(Space s, int level);
  LevelData& ref_level(Space s, int level);  // level() + reference numbering
  void ensure_p1_variant_tasks(LevelData& ld);  // K1 A/B variants' task lists

  // NCCL (one process per GPU) or loopback (virtual ranks on one GPU)
  void attach_transport(std::shared_ptr<Transport> t) { transport_ = std::move(t); }
  Transport* transport() const { return transport_.get(); }
  // interface exchange mode: false = transport send/recv (default), true =
  // direct put into the peers' receive windows; fused (put only): whether the
  // P1 stencil kernel issues the puts itself (kFusedNever, kFusedSlab: in the
  // slab partition, where it measured faster than the pack kernel,
  // kFusedAlways); set before the first level
  enum FusedPolicy { kFusedNever = 0, kFusedSlab = 1, kFusedAlways = 2 };
  void set_exchange_put(bool put, FusedPolicy fused = kFusedSlab) {
    if (!levels_.empty()) fail_arg("exchange mode: set it before the context's first level is used");
    exchange_put_ = put;
    exchange_fused_ = put ? fused : kFusedNever;
  }
  bool exchange_put() const { return exchange_put_; }
  bool exchange_fused() const {
    return exchange_fused_ == kFusedAlways || (exchange_fused_ == kFusedSlab && partition_ == kPartitionSlab);
  }

private:
  bool exchange_put_ = false;
  FusedPolicy exchange_fused_ = kFusedNever;
  MacroMesh mesh_;
  Topology topo_;
  int device_, rank_, nranks_;
  std::vector<int> macros_;
  int partition_ = kPartitionMacro;
  std::vector<int> group_;
  int ngroups_ = 0;
  cudaStream_t stream_ = nullptr;
  cudaStream_t own_stream_ = nullptr;
  cudaEvent_t switch_event_ = nullptr;
  std::map<std::pair<int, int>, std::unique_ptr<LevelData>> levels_;
  std::shared_ptr<Transport> transport_;
};

class Function {
public:
  Function(Context& ctx, Space s) : ctx_(&ctx), space_(s) {}
  Context& ctx() const { return *ctx_; }
  Space space() const { return space_; }
  double* data(int level);              // allocates (zeroed) on first use
  const double* data(int level) const;  // throws if never allocated
  bool has_level(int level) const { return data_.count(level) > 0; }
  i64 size(int level) const;            // storage entries on this rank

  void fill_seeded(int level, std::uint64_t seed, bool dirichlet_zero);
  void fill_coefficient(int level, CoeffSpec spec);
  void import_ref(int level, const double* host_ref);  // reference numbering in
  void export_ref(int level, double* host_ref);        // reference numbering out
  void import_ref_device(int level, const double* dev_ref);
  void export_ref_device(int level, double* dev_ref);
  // multi-rank I/O in reference numbering: this rank's owned slice [lo, hi)
  // (carriers whose owner macro -- the lowest sharing macro id -- is local);
  // import fills the ghost copies by the owner broadcast (collective)
  void owned_ref_range(int level, i64* lo, i64* hi);
  void import_ref_owned(int level, const double* host_owned);
  void export_ref_owned(int level, double* host_owned);
  i64 num_ref_dofs(int level);

private:
  Context* ctx_;
  Space space_;
  std::map<int, DeviceBuffer<double>> data_;
};

class Operator {
public:
  Operator(Context& ctx, Form form, std::vector<const Function*> coeffs);
  Form form() const { return form_; }
  const FormInfo& info() const { return form_info(form_); }
  void apply(const Function& src, Function& dst, int level, Update upd);
  // operator diagonal d_i = A_ii (every interface copy holds the full sum;
  // Jacobi / Chebyshev smoothing, Jacobi-preconditioned CG)
  void diagonal(Function& d, int level);

  // bench instrumentation: CUDA events around the element kernel (K1-K3)
  // on the context stream; stats() synchronizes and sums the durations.
  void set_profiling(bool on);
  void kernel_stats(double* total_ms, i64* launches);
  double* ref_scratch(i64 count);  // device buffer for reference-numbered I/O
  // 0 = optimized kernels (default), 1 = first-version kernels (k_apply_v1.cu),
  // kept selectable for A/B parity tests and the bench's history
  void set_kernel_variant(int v) { kernel_variant_ = v; }
  // integration rule of apply / diagonal: 0 = exact (default; equals the
  // reference's reference_apply), d = 1..6: the reference's quadrature(d)
  // (FormSystem::apply(v, coeffs, quadrature(d)), forms.cpp:195-255). P1 and
  // P1K are exact for every d; N1 is under-integrated for d <= 2, P2V for
  // d <= 3 ("U", forms.cpp:12)
  void set_quadrature(int degree);
  // negative control: adds delta to entry `index` of the level's
  // device table image the element kernel reads (N1 Gram table, P1 / P1K
  // stencil + stiffness table, P2V table; all geometry groups, flat double
  // index) -- a corrupted table must make parity fail
  void debug_perturb_table(int level, i64 index, double delta);
  int quadrature() const { return quad_degree_; }

private:
  // rule index of the element kernels: 0 exact, else the degree
  int rule_index() const;
  struct LevelTables {
    DeviceBuffer<P1DeviceTable> p1;
    DeviceBuffer<N1DeviceTable> n1;
    DeviceBuffer<N1GramTable> n1g;       // Gram form per geometry group (K3 v2)
    DeviceBuffer<P2VTable> p2v;          // P2V coefficient-basis tables per geometry group
  };
  LevelTables& tables(int level);
  void check(const Function& src, const Function& dst, int level) const;
  void kernel_apply(const double* x, double* y, int level);

  Context* ctx_;
  Form form_;
  std::vector<const Function*> coeffs_;
  std::map<int, std::unique_ptr<LevelTables>> tables_;
  std::map<int, DeviceBuffer<double>> scratch_;
  DeviceBuffer<double> ref_scratch_;
  bool profiling_ = false;
  int kernel_variant_ = 0;
  int quad_degree_ = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events_;
  std::size_t events_used_ = 0;
  double prof_ms_ = 0.0;
  i64 prof_launches_ = 0;

public:
  ~Operator();
};

// number of kernels this library has launched (process-wide)
i64 launch_count();

// zeroed guard entries before / after every level buffer (runtime.cpp)
i64 storage_guard(int n);

// default contiguous partition of macro ids over ranks
std::vector<int> partition_macros(int num_macros, int rank, int nranks);

} // namespace tetmf
