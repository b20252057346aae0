// gs_torch_ops.cpp — the hot-path entry points of libgearserve_b200.so as
// torch operators (TORCH_LIBRARY namespace gearserve_b200), so they go
// through the dispatcher: torch.ops.gearserve_b200.<op>(...) on CUDA tensors,
// outputs from the caching allocator, launched on the current stream.
//
// Thin: each op checks shapes / dtypes / devices, allocates its outputs and
// workspace, and calls the C ABI (include/gearserve_b200.h), whose codes map
// to the reference's exceptions (GS_EINVAL -> ValueError, GS_EUNSUPPORTED ->
// ValueError naming the limit, anything else -> RuntimeError).  The numpy
// surface of the reference (kernels.evaluate_encoded etc.) stays in the
// Python package; these ops are its tensor-level equivalents:
//   evaluate_encoded  src/kernels.py:93-108  (gs_eval_encoded)
//   grid_sweep        the full cascade x ThresholdGrid product
//                     (src/cascades.py:132-193; gs_grid_plan/build/eval)
//   pareto_counts     cascades.pareto_filter on integer counts (src/cascades.py:116-129)
//   certainty         cascades.certainty per row (src/cascades.py:20-28)
//   quantiles         np.quantile(column, qs) for build_threshold_grid (src/cascades.py:150-163)
//   head_certainty    a stage's classifier head + certainty on the tensor cores (gs_head.cu)
#include <ATen/ATen.h>
#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGuard.h>
#include <torch/library.h>

#include <string>
#include <tuple>
#include <vector>

#include "gearserve_b200.h"

namespace {

void check_rc(int rc, const char* what) {
  if (rc == GS_OK) return;
  const std::string msg = std::string(what) + ": " + gs_strerror(rc) +
                          (rc == GS_ECUDA ? std::string(" (") + gs_last_cuda_error() + ")" : "");
  TORCH_CHECK_VALUE(rc != GS_EINVAL && rc != GS_EUNSUPPORTED, msg);
  TORCH_CHECK(false, msg);
}

void* cur_stream() { return static_cast<void*>(at::cuda::getCurrentCUDAStream().stream()); }

at::Tensor dev_contig(const at::Tensor& t, at::ScalarType dt, const at::Device& dev, const char* name) {
  TORCH_CHECK_VALUE(t.device() == dev, name, " must be on ", dev, ", got ", t.device());
  TORCH_CHECK_VALUE(t.scalar_type() == dt, name, " must be ", dt, ", got ", t.scalar_type());
  return t.contiguous();
}

at::Tensor workspace(size_t bytes, const at::Device& dev) {
  return at::empty({(int64_t)std::max<size_t>(bytes, 1)}, at::TensorOptions().dtype(at::kByte).device(dev));
}

std::tuple<at::Tensor, at::Tensor, at::Tensor> evaluate_encoded(const at::Tensor& certainty,
                                                                const at::Tensor& correct,
                                                                const at::Tensor& stage_model,
                                                                const at::Tensor& thresholds,
                                                                const at::Tensor& n_stages,
                                                                const at::Tensor& cost1) {
  TORCH_CHECK_VALUE(certainty.dim() == 2 && correct.sizes() == certainty.sizes(),
                    "certainty and correct must be matching [n_rec, n_models] matrices");
  TORCH_CHECK_VALUE(stage_model.dim() == 2 && thresholds.sizes() == stage_model.sizes(),
                    "stage_model and thresholds must be matching [n_casc, max_len] matrices");
  const at::Device dev = certainty.device();
  TORCH_CHECK_VALUE(dev.is_cuda(), "certainty must be a CUDA tensor");
  const c10::cuda::CUDAGuard guard(dev);
  const auto cert = dev_contig(certainty, at::kDouble, dev, "certainty");
  const auto corr = dev_contig(correct, at::kByte, dev, "correct");
  const auto sm = dev_contig(stage_model, at::kInt, dev, "stage_model");
  const auto thr = dev_contig(thresholds, at::kDouble, dev, "thresholds");
  const auto ns = dev_contig(n_stages, at::kInt, dev, "n_stages");
  const auto c1 = dev_contig(cost1, at::kDouble, dev, "cost1");
  const int64_t n_rec = cert.size(0), n_casc = sm.size(0);
  const int32_t M = (int32_t)cert.size(1), L = (int32_t)sm.size(1);
  TORCH_CHECK_VALUE(ns.numel() == n_casc && c1.numel() == M, "n_stages / cost1 lengths");
  const auto opt = cert.options();
  auto acc = at::empty({n_casc}, opt), cost = at::empty({n_casc}, opt), frac = at::empty({n_casc, L}, opt);
  size_t bytes = 0;
  check_rc(gs_eval_encoded_workspace(n_rec, M, n_casc, L, &bytes), "evaluate_encoded");
  auto ws = workspace(bytes, dev);
  check_rc(gs_eval_encoded(cert.data_ptr<double>(), corr.data_ptr<uint8_t>(), n_rec, M, sm.data_ptr<int32_t>(),
                           thr.data_ptr<double>(), ns.data_ptr<int32_t>(), n_casc, L, c1.data_ptr<double>(),
                           acc.data_ptr<double>(), cost.data_ptr<double>(), frac.data_ptr<double>(),
                           ws.data_ptr(), ws.numel(), cur_stream()),
           "evaluate_encoded");
  return {acc, cost, frac};
}

std::tuple<at::Tensor, at::Tensor, at::Tensor, at::Tensor> grid_sweep(const at::Tensor& certainty,
                                                                      const at::Tensor& correct,
                                                                      const at::Tensor& grids,
                                                                      at::IntArrayRef grid_len,
                                                                      const at::Tensor& cost1) {
  TORCH_CHECK_VALUE(certainty.dim() == 2 && correct.sizes() == certainty.sizes(),
                    "certainty and correct must be matching [n_rec, n_models] matrices");
  const at::Device dev = certainty.device();
  TORCH_CHECK_VALUE(dev.is_cuda(), "certainty must be a CUDA tensor");
  const c10::cuda::CUDAGuard guard(dev);
  const auto cert = dev_contig(certainty, at::kDouble, dev, "certainty");
  const auto corr = dev_contig(correct, at::kByte, dev, "correct");
  const auto g = dev_contig(grids, at::kDouble, dev, "grids");
  const auto c1 = dev_contig(cost1, at::kDouble, dev, "cost1");
  const int64_t n_rec = cert.size(0);
  const int32_t M = (int32_t)cert.size(1);
  TORCH_CHECK_VALUE((int64_t)grid_len.size() == M && c1.numel() == M, "grid_len / cost1 need one entry per model");
  std::vector<int32_t> gl(grid_len.begin(), grid_len.end());
  int64_t total = 0;
  for (int32_t v : gl) total += v;
  TORCH_CHECK_VALUE(g.numel() == total, "grids must hold sum(grid_len) values");
  gs_grid_info info{};
  check_rc(gs_grid_plan(n_rec, M, gl.data(), &info), "grid_sweep");
  auto ws = workspace(info.workspace_bytes, dev);
  void* st = cur_stream();
  check_rc(gs_grid_build(cert.data_ptr<double>(), corr.data_ptr<uint8_t>(), n_rec, M, g.data_ptr<double>(),
                         gl.data(), ws.data_ptr(), ws.numel(), GS_GRID_WORKSPACE_DIRTY, st),
           "grid_sweep");
  const auto opt = cert.options();
  const int64_t C = info.n_configs;
  auto acc = at::empty({C}, opt), cost = at::empty({C}, opt), frac = at::empty({C, info.max_len}, opt);
  auto nc = at::empty({C}, opt.dtype(at::kInt));
  check_rc(gs_grid_eval(n_rec, M, gl.data(), c1.data_ptr<double>(), 0, C, acc.data_ptr<double>(),
                        cost.data_ptr<double>(), frac.data_ptr<double>(),
                        reinterpret_cast<uint32_t*>(nc.data_ptr<int32_t>()), ws.data_ptr(), ws.numel(), st),
           "grid_sweep");
  return {acc, cost, frac, nc};
}

at::Tensor pareto_counts(const at::Tensor& n_correct, const at::Tensor& mean_cost, int64_t n_rec) {
  const at::Device dev = n_correct.device();
  TORCH_CHECK_VALUE(dev.is_cuda(), "n_correct must be a CUDA tensor");
  const c10::cuda::CUDAGuard guard(dev);
  const auto nc = dev_contig(n_correct, at::kInt, dev, "n_correct");
  const auto cost = dev_contig(mean_cost, at::kDouble, dev, "mean_cost");
  const int64_t n = nc.numel();
  TORCH_CHECK_VALUE(cost.numel() == n, "n_correct and mean_cost lengths differ");
  size_t bytes = 0;
  check_rc(gs_pareto_counts_workspace(n, n_rec, &bytes), "pareto_counts");
  auto ws = workspace(bytes, dev);
  auto keep = at::empty({std::max<int64_t>(n, 1)}, nc.options().dtype(at::kByte));
  auto idx = at::empty({std::max<int64_t>(n, 1)}, nc.options().dtype(at::kLong));
  auto cnt = at::empty({1}, nc.options().dtype(at::kLong));
  check_rc(gs_pareto_counts(reinterpret_cast<const uint32_t*>(nc.data_ptr<int32_t>()), cost.data_ptr<double>(), n,
                            n_rec, 0, keep.data_ptr<uint8_t>(), idx.data_ptr<int64_t>(), cnt.data_ptr<int64_t>(),
                            ws.data_ptr(), ws.numel(), cur_stream()),
           "pareto_counts");
  return idx.narrow(0, 0, cnt.item<int64_t>());  // the kept indices, ascending
}

at::Tensor certainty(const at::Tensor& scores, int64_t kind) {
  TORCH_CHECK_VALUE(scores.dim() == 2, "scores must be [n_rows, n_cls]");
  const at::Device dev = scores.device();
  TORCH_CHECK_VALUE(dev.is_cuda(), "scores must be a CUDA tensor");
  const c10::cuda::CUDAGuard guard(dev);
  int32_t dt;
  switch (scores.scalar_type()) {
    case at::kFloat: dt = GS_F32; break;
    case at::kDouble: dt = GS_F64; break;
    case at::kBFloat16: dt = GS_BF16; break;
    default: TORCH_CHECK_VALUE(false, "scores must be float32, float64 or bfloat16");
  }
  const auto s = scores.stride(1) == 1 ? scores : scores.contiguous();
  auto out = at::empty({s.size(0)}, s.options().dtype(at::kDouble));
  check_rc(gs_certainty(s.data_ptr(), dt, s.size(0), (int32_t)s.size(1), s.stride(0), nullptr, (int32_t)kind,
                        out.data_ptr<double>(), cur_stream()),
           "certainty");
  return out;
}

at::Tensor quantiles(const at::Tensor& column, at::ArrayRef<double> qs) {
  TORCH_CHECK_VALUE(column.dim() == 1 && column.numel() > 0, "quantiles of an empty or non-1-D column");
  const at::Device dev = column.device();
  TORCH_CHECK_VALUE(dev.is_cuda(), "column must be a CUDA tensor");
  const c10::cuda::CUDAGuard guard(dev);
  TORCH_CHECK_VALUE(column.scalar_type() == at::kDouble, "column must be float64");  // any stride
  const std::vector<double> q(qs.begin(), qs.end());
  size_t bytes = 0;
  check_rc(gs_quantiles_workspace(column.numel(), (int32_t)q.size(), &bytes), "quantiles");
  auto ws = workspace(bytes, dev);
  auto out = at::empty({std::max<int64_t>((int64_t)q.size(), 1)}, column.options());
  check_rc(gs_quantiles(column.data_ptr<double>(), column.numel(), column.stride(0), q.data(), (int32_t)q.size(),
                        out.data_ptr<double>(), ws.data_ptr(), ws.numel(), cur_stream()),
           "quantiles");
  return out.narrow(0, 0, (int64_t)q.size());
}

at::Tensor head_certainty(const at::Tensor& features, const at::Tensor& weight, const c10::optional<at::Tensor>& bias,
                          int64_t kind) {
  TORCH_CHECK_VALUE(features.dim() == 2 && weight.dim() == 2 && features.size(1) == weight.size(1),
                    "features [B, K] and weight [N, K] must share K");
  const at::Device dev = features.device();
  TORCH_CHECK_VALUE(dev.is_cuda(), "features must be a CUDA tensor");
  const c10::cuda::CUDAGuard guard(dev);
  const auto f = dev_contig(features, at::kBFloat16, dev, "features");
  const auto w = dev_contig(weight, at::kBFloat16, dev, "weight");
  at::Tensor b;
  if (bias.has_value()) {
    b = dev_contig(*bias, at::kFloat, dev, "bias");
    TORCH_CHECK_VALUE(b.numel() == w.size(0), "bias must hold one value per class");
  }
  auto cert = at::empty({f.size(0)}, f.options().dtype(at::kDouble));
  check_rc(gs_head_certainty(f.data_ptr(), w.data_ptr(), b.defined() ? b.data_ptr<float>() : nullptr, f.size(0),
                             (int32_t)w.size(0), (int32_t)f.size(1), (int32_t)kind, cert.data_ptr<double>(), nullptr,
                             cur_stream()),
           "head_certainty");
  return cert;
}

}  // namespace

TORCH_LIBRARY(gearserve_b200, m) {
  m.def("evaluate_encoded(Tensor certainty, Tensor correct, Tensor stage_model, Tensor thresholds, "
        "Tensor n_stages, Tensor cost1) -> (Tensor accuracy, Tensor mean_cost, Tensor forward_frac)");
  m.def("grid_sweep(Tensor certainty, Tensor correct, Tensor grids, int[] grid_len, Tensor cost1) -> "
        "(Tensor accuracy, Tensor mean_cost, Tensor forward_frac, Tensor n_correct)");
  m.def("pareto_counts(Tensor n_correct, Tensor mean_cost, int n_rec) -> Tensor");
  m.def("certainty(Tensor scores, int kind=0) -> Tensor");
  m.def("quantiles(Tensor column, float[] qs) -> Tensor");
  m.def("head_certainty(Tensor features, Tensor weight, Tensor? bias=None, int kind=2) -> Tensor");
}

TORCH_LIBRARY_IMPL(gearserve_b200, CUDA, m) {
  m.impl("evaluate_encoded", &evaluate_encoded);
  m.impl("grid_sweep", &grid_sweep);
  m.impl("pareto_counts", &pareto_counts);
  m.impl("certainty", &certainty);
  m.impl("quantiles", &quantiles);
  m.impl("head_certainty", &head_certainty);
}
