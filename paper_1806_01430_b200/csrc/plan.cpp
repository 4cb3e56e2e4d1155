// plan.cpp -- the device-residency planner.
//
// The paper's offload killer is the implicit copy of every touched array around every
// `kernels` region.  Here each array carries a validity state
// {host, device}; a transfer is emitted only when a nest reads an array on a side where
// it is not valid, and a write invalidates the other side.  Data flow of the program
// (fixtures/matmul.c:8-34):
//   a : init-a -> matmul        b : init-b -> transpose      bt : transpose -> matmul
//   c : zero-c -> matmul -> trace                            sum: trace -> printf (host)
#include "plan.hpp"

#include <cstring>

namespace mmx {

const LoopRow kCatalogue[MMX_GENE_LENGTH] = {
    {0, 8, 0, MMX_NEST_INIT_A, "i", "fill2d<init_a>"},
    {1, 9, 1, MMX_NEST_INIT_A, "j", "fill_row<init_a>"},
    {2, 12, 0, MMX_NEST_INIT_B, "i", "fill2d<init_b>"},
    {3, 13, 1, MMX_NEST_INIT_B, "j", "fill_row<init_b>"},
    {4, 16, 0, MMX_NEST_ZERO_C, "i", "fill2d<zero>"},
    {5, 17, 1, MMX_NEST_ZERO_C, "j", "fill_row<zero>"},
    {6, 21, 0, MMX_NEST_TRANSPOSE, "i", "transpose_tiled"},
    {7, 22, 1, MMX_NEST_TRANSPOSE, "j", "transpose_row_gather"},
    {8, 25, 0, MMX_NEST_MATMUL, "i", "matmul_nt"},
    {9, 26, 1, MMX_NEST_MATMUL, "j", "gemv_row"},
    {10, 27, 2, MMX_NEST_MATMUL, "k", "dot_rows"},
    {11, 31, 0, MMX_NEST_TRACE, "i", "trace_diag"},
};

const NestRow kNests[MMX_NUM_NESTS] = {{0, 2}, {2, 2}, {4, 2}, {6, 2}, {8, 3}, {11, 1}};

namespace {

struct Residency {
  bool host = false, device = false;
};

struct Builder {
  mmx_plan_info* p;
  std::uint64_t matrix_bytes, elem_bytes, n;
  Residency arr[MMX_NUM_ARRAYS];

  void push(int kind, int nest, int array, int mode, std::uint64_t bytes, std::uint64_t launches) {
    if (p->num_steps >= MMX_MAX_PLAN_STEPS) return;
    mmx_plan_step& s = p->steps[p->num_steps++];
    s.kind = kind;
    s.nest = nest;
    s.array = array;
    s.mode = mode;
    s.bytes = bytes;
    s.launches = launches;
    if (kind == MMX_STEP_H2D || kind == MMX_STEP_H2D_DIAG) p->h2d_bytes += bytes;
    if (kind == MMX_STEP_D2H || kind == MMX_STEP_D2H_DIAG || kind == MMX_STEP_D2H_SUM) p->d2h_bytes += bytes;
    p->kernel_launches += launches;
  }

  // make `array` readable on the given side
  void need(int array, bool on_device) {
    Residency& r = arr[array];
    if (on_device && !r.device) {
      push(MMX_STEP_H2D, -1, array, -1, matrix_bytes, 0);
      r.device = true;
    } else if (!on_device && !r.host) {
      push(MMX_STEP_D2H, -1, array, -1, matrix_bytes, 0);
      r.host = true;
    }
  }
  void wrote(int array, bool on_device) {
    arr[array].device = on_device;
    arr[array].host = !on_device;
  }
};

std::uint64_t launches_of(int mode, std::uint64_t n) {
  switch (mode) {
    case MMX_MODE_GPU_NEST: return 1;
    case MMX_MODE_GPU_INNER: return n;
    case MMX_MODE_GPU_INNER2: return n * n;
    default: return 0;
  }
}

}  // namespace

int build_plan(const std::uint8_t* bits, std::size_t gene_len, std::int32_t n, std::int32_t dtype,
               mmx_plan_info* out) {
  if (out == nullptr || bits == nullptr) return MMX_E_INVALID;
  if (gene_len != MMX_GENE_LENGTH) return MMX_E_LENGTH;
  if (n < 1 || (dtype != MMX_F64 && dtype != MMX_F32)) return MMX_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  out->feasible = 1;
  out->conflict_nest = -1;

  // One annotated loop per nest at most: a second one would sit inside the first one's
  // compute region ("compute regions may not be nested").
  for (int nest = 0; nest < MMX_NUM_NESTS; ++nest) {
    int set = 0, mode = MMX_MODE_CPU;
    for (int d = 0; d < kNests[nest].depth_count; ++d) {
      if (bits[kNests[nest].first_gene + d] != 0) {
        ++set;
        mode = MMX_MODE_GPU_NEST + d;
      }
    }
    out->modes[nest] = mode;
    if (set > 1 && out->feasible) {
      out->feasible = 0;
      out->conflict_nest = nest;
    }
  }
  if (!out->feasible) return MMX_OK;

  Builder b;
  b.p = out;
  b.n = static_cast<std::uint64_t>(n);
  b.elem_bytes = elem_size(dtype);
  b.matrix_bytes = b.n * b.n * b.elem_bytes;

  auto run = [&](int nest) {
    const int mode = out->modes[nest];
    const bool dev = mode != MMX_MODE_CPU;
    b.push(dev ? MMX_STEP_GPU : MMX_STEP_CPU, nest, -1, mode, 0, launches_of(mode, b.n));
    return dev;
  };

  b.wrote(MMX_ARRAY_A, run(MMX_NEST_INIT_A));
  b.wrote(MMX_ARRAY_B, run(MMX_NEST_INIT_B));
  b.wrote(MMX_ARRAY_C, run(MMX_NEST_ZERO_C));

  {
    const bool dev = out->modes[MMX_NEST_TRANSPOSE] != MMX_MODE_CPU;
    b.need(MMX_ARRAY_B, dev);
    b.wrote(MMX_ARRAY_BT, run(MMX_NEST_TRANSPOSE));
  }
  {
    const bool dev = out->modes[MMX_NEST_MATMUL] != MMX_MODE_CPU;
    b.need(MMX_ARRAY_A, dev);
    b.need(MMX_ARRAY_BT, dev);
    b.need(MMX_ARRAY_C, dev);
    b.wrote(MMX_ARRAY_C, run(MMX_NEST_MATMUL));
  }
  {
    const bool dev = out->modes[MMX_NEST_TRACE] != MMX_MODE_CPU;
    // the trace reads only c[i][i]: move the diagonal (strided 2-D copy), not the matrix
    if (dev) {
      if (!b.arr[MMX_ARRAY_C].device) b.push(MMX_STEP_H2D_DIAG, -1, MMX_ARRAY_C, -1, b.n * b.elem_bytes, 0);
      run(MMX_NEST_TRACE);
      b.push(MMX_STEP_D2H_SUM, -1, -1, -1, b.elem_bytes, 0);
    } else {
      if (!b.arr[MMX_ARRAY_C].host) b.push(MMX_STEP_D2H_DIAG, -1, MMX_ARRAY_C, -1, b.n * b.elem_bytes, 0);
      run(MMX_NEST_TRACE);
    }
  }

  // Lower bound, derived independently of the state machine above: one term per
  // producer->consumer edge of the data-flow graph whose ends sit on different sides, each
  // sized by what the consumer reads.
  struct Edge {
    int producer, consumer;
    bool diagonal_only;
  };
  static const Edge kEdges[] = {
      {MMX_NEST_INIT_A, MMX_NEST_MATMUL, false},   // a
      {MMX_NEST_INIT_B, MMX_NEST_TRANSPOSE, false},  // b
      {MMX_NEST_TRANSPOSE, MMX_NEST_MATMUL, false},  // bt
      {MMX_NEST_ZERO_C, MMX_NEST_MATMUL, false},     // c (read-modify-write)
      {MMX_NEST_MATMUL, MMX_NEST_TRACE, true},       // c diagonal
  };
  for (const Edge& e : kEdges) {
    const bool pdev = out->modes[e.producer] != MMX_MODE_CPU;
    const bool cdev = out->modes[e.consumer] != MMX_MODE_CPU;
    if (pdev == cdev) continue;
    const std::uint64_t bytes = e.diagonal_only ? b.n * b.elem_bytes : b.matrix_bytes;
    (cdev ? out->h2d_lower_bound : out->d2h_lower_bound) += bytes;
  }
  if (out->modes[MMX_NEST_TRACE] != MMX_MODE_CPU) out->d2h_lower_bound += b.elem_bytes;  // sum -> printf
  return MMX_OK;
}

}  // namespace mmx
