// GPU measurements of the planner's inputs, with the reference's own
// definitions: T(B) = seconds of one transformer block's S-Part
// (project_qkv + finish_block of layer 0) at batch B (bench_dense_block,
// dense.cpp:145-196), and R = seconds of attend per token-position per layer
// (bench_attention_per_token, attention.cpp:307-354). Device-timed with CUDA
// events; each sample is an inner loop of >= 2 ms, the median of the samples
// is reported (the reference's calibration).
#include "perf_bench.h"

#include <algorithm>
#include <vector>

#include "dense_kernels.cuh"

namespace sd {

namespace {

template <typename F>
double median_seconds(F&& once, int reps, cudaStream_t s) {
  cudaEvent_t e0, e1;
  SD_CUDA(cudaEventCreate(&e0));
  SD_CUDA(cudaEventCreate(&e1));
  auto timed = [&](int inner) {
    SD_CUDA(cudaEventRecord(e0, s));
    for (int i = 0; i < inner; ++i) once();
    SD_CUDA(cudaEventRecord(e1, s));
    SD_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    return ms / 1e3;
  };
  once();  // warm-up (tensor maps, plans)
  int inner = 1;
  while (timed(inner) < 2e-3 && inner < (1 << 16)) inner *= 4;
  std::vector<double> samples;
  for (int r = 0; r < reps; ++r) samples.push_back(timed(inner) / inner);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::sort(samples.begin(), samples.end());
  return samples[samples.size() / 2];
}

}  // namespace

void bench_dense_block(Weights& w, const int* batches, int n, int reps, double* seconds) {
  if (n < 1) fail(SD_ERR_CONFIG, "bench: no batch sizes given");
  if (!std::is_sorted(batches, batches + n)) fail(SD_ERR_CONFIG, "bench: batch sizes must be ascending");
  if (reps < 1) fail(SD_ERR_CONFIG, "need at least one repetition");
  if (batches[0] < 1) fail(SD_ERR_CONFIG, "bench: batch sizes must be positive");
  DeviceGuard dg(w.device());
  const Spec& sp = w.spec();
  const size_t bmax = (static_cast<size_t>(batches[n - 1]) + 127) / 128 * 128;
  const bool bf = w.mode() == SD_DENSE_BF16 || w.mode() == SD_DENSE_F16;
  const int f16 = w.mode() == SD_DENSE_F16 ? 1 : 0;
  DevBuf x, qkv, y, h, xo, xb, ob, yb, hb;
  const size_t D = sp.D, F = sp.F, Q = sp.qkv_width();
  for (auto* b : {&x, &y, &xo}) SD_CUDA(cudaMemset(b->get(bmax * D * 4), 0, bmax * D * 4));
  SD_CUDA(cudaMemset(qkv.get(bmax * Q * 4), 0, bmax * Q * 4));
  SD_CUDA(cudaMemset(h.get(bmax * F * 4), 0, bmax * F * 4));
  for (auto* b : {&xb, &ob, &yb}) SD_CUDA(cudaMemset(b->get(bmax * D * 2), 0, bmax * D * 2));
  SD_CUDA(cudaMemset(hb.get(bmax * F * 2), 0, bmax * F * 2));
  SD_CUDA(cudaDeviceSynchronize());
  cudaStream_t s;
  SD_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // data-dependent tensor-core power: the features are random values (the
  // reference feeds deterministic_batch features, dense.cpp:145-196), not zeros
  launch_fill_synthetic(static_cast<float*>(x.p), static_cast<int64_t>(bmax * D), 0xB0B5ull, s);
  if (bf) launch_to_16(static_cast<int>(bmax), static_cast<int>(D), static_cast<float*>(x.p), D, xb.p, D,
                       w.mode() == SD_DENSE_F16, s);
  SD_CUDA(cudaStreamSynchronize(s));
  auto f = [](DevBuf& b) { return static_cast<float*>(b.p); };
  auto hbf = [](DevBuf& b) { return static_cast<act16*>(b.p); };
  for (int i = 0; i < n; ++i) {
    const int B = batches[i];
    // project_qkv + finish_block of layer 0 (the reference's run_once); the
    // attention output o is taken as the q block as in the reference
    auto once = [&] {
      w.linear(0, 0, B, f(x), D, hbf(xb), D, f(qkv), Q, nullptr, 0, kEpiNone, nullptr, 0, s);
      if (bf) launch_to_16(B, static_cast<int>(D), f(qkv), Q, hbf(ob), D, f16, s);
      w.linear(0, 4, B, f(qkv), Q, hbf(ob), D, f(y), D, bf ? hbf(yb) : nullptr, D, kEpiResidual, f(x), D, s);
      w.linear(0, 5, B, f(y), D, hbf(yb), D, bf ? nullptr : f(h), F, bf ? hbf(hb) : nullptr, F, kEpiSilu, nullptr, 0, s);
      w.linear(0, 6, B, f(h), F, hbf(hb), F, f(xo), D, nullptr, 0, kEpiResidual, f(y), D, s);
    };
    seconds[i] = median_seconds(once, reps, s);
  }
  SD_CUDA(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
}

double bench_attention_per_token(const Spec& spec, int fmt, int batch, int seq_len, int reps, int device) {
  if (reps < 1) fail(SD_ERR_CONFIG, "need at least one repetition");
  if (batch < 1 || seq_len < 1) fail(SD_ERR_CONFIG, "bench: batch and sequence length must be >= 1");
  DeviceGuard dg(device);
  sd_kv_options o{};
  o.max_sequences = batch;
  o.max_seq_len = seq_len + 1;
  KvStore kv(spec, 0, spec.Hkv, static_cast<int64_t>(batch) * seq_len + batch, fmt, device, &o);
  std::vector<uint64_t> seqs(static_cast<size_t>(batch));
  for (int b = 0; b < batch; ++b) seqs[static_cast<size_t>(b)] = static_cast<uint64_t>(b + 1);
  cudaStream_t s;
  SD_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  kv.prefill_synthetic(batch, seqs.data(), seq_len, 42, s);
  DevBuf q, out;
  const size_t qw = static_cast<size_t>(kv.q_width());
  SD_CUDA(cudaMemsetAsync(q.get(static_cast<size_t>(batch) * qw * 4), 0, static_cast<size_t>(batch) * qw * 4, s));
  out.get(static_cast<size_t>(batch) * qw * 4);
  auto once = [&] {
    kv.attend(0, batch, seqs.data(), static_cast<float*>(q.p), static_cast<int64_t>(qw), static_cast<float*>(out.p),
              static_cast<int64_t>(qw), s);
  };
  const double t = median_seconds(once, reps, s);
  SD_CUDA(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
  return t / (static_cast<double>(batch) * seq_len);
}

int64_t kv_capacity_tokens(const Spec& spec, int fmt, int device, double reserve_bytes) {
  DeviceGuard dg(device);
  size_t free_b = 0, total_b = 0;
  SD_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double w = static_cast<double>(spec.kv_width());
  const double per_pos = fmt == SD_KV_SINGLE ? 2 * w * 4 : fmt == SD_KV_HALF ? 2 * w * 2 : 2 * (w + spec.Hkv * 4.0);
  const double usable = static_cast<double>(free_b) - reserve_bytes;
  return usable > 0 ? static_cast<int64_t>(usable / (per_pos * spec.L)) : 0;
}

}  // namespace sd
