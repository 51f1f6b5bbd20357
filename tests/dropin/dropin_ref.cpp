// dropin_ref.cpp -- GPU actors from libdf_cuda.so running INSIDE the
// reference's own runtime (dynflow::run, thread per actor), as
// INTEGRATION.md §2 describes.  Test infrastructure: compiled against the
// reference headers (/root/reference/proj/include) and linked with the
// reference compiled from its sources (oracle/_ref/libdynflow_ref.so) and
// with libdf_cuda.so; the binary lands in oracle/_ref/ (built here, run on
// the GPU box by tests/test_dropin_ref_gpu.py).
//
// Cases (each prints PASS/FAIL <name>):
//   motion_r{1,4}  source -> motion_gpu -> sink: gauss/thres/med replaced by
//                  ONE GPU actor behind dynflow::bulk_kernel_adapter
//                  (runtime.hpp:97-108); byte-equal to the reference's own
//                  oracle_motion_detection_raw on acceptance [6]'s input
//                  (64 frames 320x240, seed 606) at token rate 1 and 4.
//   dpd_acc8       source -> config -> dpd_gpu (dynamic: its control
//                  function is the reference's check_config, rates 1) ->
//                  sink: split / 10 branches / adder replaced by ONE GPU
//                  actor calling df_dpd_fire; bit-equal to the reference's
//                  oracle_dpd on acceptance [8] (2^20, period 65536, taps
//                  808, schedule (16, 809), input 810).
//   dpd_p4096      the same on a period-4096 random schedule (seed 2020).
//   fault          a GPU actor whose C-ABI call fails (DF_EINVAL) ends run() with
//                  ActorFault naming it (runtime.cpp:232-247).
#include <complex>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "df_cuda.h"
#include "dynflow/dpd.hpp"
#include "dynflow/model.hpp"
#include "dynflow/motion.hpp"
#include "dynflow/runtime.hpp"

using namespace dynflow;

namespace {

void ck(int rc) {
  if (rc != DF_OK) throw std::runtime_error(std::string("df_cuda: ") + df_last_error());
}

int failures = 0;
void report(const std::string& name, bool ok, const std::string& why = "") {
  std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), why.empty() ? "" : " ", why.c_str());
  std::fflush(stdout);
  if (!ok) ++failures;
}

// ---- motion: one GPU actor behind bulk_kernel_adapter --------------------
struct GpuMotion {
  df_motion* m = nullptr;
  void* stream = nullptr;
  void* in = nullptr;
  void* out = nullptr;
  std::size_t frame = 0;
  GpuMotion(unsigned w, unsigned h, std::uint8_t thr, std::uint32_t rate) : frame(std::size_t(w) * h) {
    ck(df_motion_create(0, w, h, DF_MOTION_GRAY, thr, &m));
    ck(df_stream_create(0, &stream));
    ck(df_malloc(0, frame * rate, &in));
    ck(df_malloc(0, frame * rate, &out));
  }
  ~GpuMotion() {
    df_free(in);
    df_free(out);
    df_stream_destroy(stream);
    df_motion_destroy(m);
  }
};

std::vector<std::uint8_t> run_motion_dropin(const std::vector<std::uint8_t>& frames, unsigned w, unsigned h,
                                            std::uint8_t thr, std::uint32_t r, bool inject_fault = false) {
  const std::size_t size = std::size_t(w) * h;
  const std::uint64_t nframes = frames.size() / size;
  std::vector<std::uint8_t> output(frames.size());
  std::vector<ChannelSpec> channels = {{"src_gpu", size, r, false, {}}, {"gpu_sink", size, r, false, {}}};
  ActorBehavior source;  // motion.cpp:123-129
  const std::uint8_t* in = frames.data();
  source.fire = [in, size](FiringContext& ctx) {
    auto region = ctx.output(0);
    std::memcpy(region.data(), in + ctx.firing_index() * ctx.output_tokens(0) * size, region.size());
  };
  auto gpu = std::make_shared<GpuMotion>(w, h, thr, r);
  // gauss + thres + med as ONE device kernel; the one-frame delay token
  // (gauss of the previous frame, black first) lives inside the actor.
  ActorBehavior motion_gpu = bulk_kernel_adapter([gpu, r, inject_fault](const std::vector<std::span<const std::byte>>& ins) {
    const std::size_t bytes = ins[0].size();
    ck(df_memcpy_h2d(gpu->in, ins[0].data(), bytes, gpu->stream));
    ck(df_motion_fire(gpu->m, gpu->in, inject_fault ? nullptr : static_cast<std::uint8_t*>(gpu->out), r, gpu->stream));
    std::vector<std::vector<std::byte>> outs(1, std::vector<std::byte>(bytes));
    ck(df_memcpy_d2h(outs[0].data(), gpu->out, bytes, gpu->stream));
    ck(df_stream_synchronize(gpu->stream));
    return outs;
  });
  ActorBehavior sink;  // motion.cpp:178-183
  std::uint8_t* outp = output.data();
  sink.fire = [outp, size](FiringContext& ctx) {
    auto region = ctx.input(0);
    std::memcpy(outp + ctx.firing_index() * ctx.input_tokens(0) * size, region.data(), region.size());
  };
  std::vector<ActorSpec> actors = {
      {"source", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "src_gpu"}}, source, {}},
      {"motion_gpu",
       ActorKind::static_rate,
       {{PortDirection::input, PortKind::regular, "src_gpu"}, {PortDirection::output, PortKind::regular, "gpu_sink"}},
       motion_gpu,
       {}},
      {"sink", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "gpu_sink"}}, sink, {}},
  };
  ExecutionConfig cfg;
  cfg.source_firing_limit = nframes / r;
  run(build_network(actors, channels), cfg);
  return output;
}

// ---- DPD: one dynamic GPU actor replacing split / branches / adder -------
struct GpuDpd {
  df_dpd* d = nullptr;
  void* stream = nullptr;
  void *ctrl = nullptr, *in = nullptr, *out = nullptr;
  std::vector<float> host;  // interleaved staging
  std::uint32_t token = 0;  // set by control, read by fire (same actor thread)
  GpuDpd(std::uint32_t period, const dpd::TapSet& taps) : host(2ull * period) {
    std::vector<float> flat;
    for (const auto& br : taps)
      for (const auto& t : br) {
        flat.push_back(t.real());
        flat.push_back(t.imag());
      }
    ck(df_dpd_create(0, period, 10, flat.data(), &d));
    ck(df_stream_create(0, &stream));
    ck(df_malloc(0, 4, &ctrl));
    ck(df_malloc(0, 8ull * period, &in));
    ck(df_malloc(0, 8ull * period, &out));
  }
  ~GpuDpd() {
    df_free(ctrl);
    df_free(in);
    df_free(out);
    df_stream_destroy(stream);
    df_dpd_destroy(d);
  }
};

std::vector<std::complex<float>> run_dpd_dropin(const dpd::Params& p) {
  const std::uint32_t period = p.period;
  const std::size_t plane = std::size_t(period) * sizeof(float);
  std::vector<std::complex<float>> output(p.samples);
  std::vector<ChannelSpec> channels = {{"src_re", plane, 1, false, {}},  {"src_im", plane, 1, false, {}},
                                       {"gpu_re", plane, 1, false, {}},  {"gpu_im", plane, 1, false, {}},
                                       {"cfg_gpu", dpd::kConfigTokenBytes, 1, false, {}}};
  const auto input = p.input;
  ActorBehavior source;  // dpd.cpp:189-204
  source.fire = [input, period](FiringContext& ctx) {
    auto* re = reinterpret_cast<float*>(ctx.output(0).data());
    auto* im = reinterpret_cast<float*>(ctx.output(1).data());
    const std::size_t base = ctx.firing_index() * period;
    for (std::size_t i = 0; i < period; ++i) {
      re[i] = input[base + i].real();
      im[i] = input[base + i].imag();
    }
  };
  const auto schedule = p.schedule;
  ActorBehavior config;  // dpd.cpp:206-221
  config.fire = [schedule](FiringContext& ctx) {
    dpd::encode_config(schedule[ctx.firing_index() % schedule.size()], ctx.output(0));
  };
  auto gpu = std::make_shared<GpuDpd>(period, p.taps);
  ActorBehavior dpd_gpu;
  dpd_gpu.control = [gpu](std::span<const std::byte> token) {
    const dpd::ConfigToken t = dpd::decode_config(token);
    dpd::check_config(t);  // dpd.cpp:49-58 -> ControlError path via ActorFault
    gpu->token = t.active_mask;
    return FiringRates::uniform(4, 1);  // the block goes in and out every firing; gating is on the device
  };
  dpd_gpu.fire = [gpu, period](FiringContext& ctx) {
    const float* re = reinterpret_cast<const float*>(ctx.input(0).data());
    const float* im = reinterpret_cast<const float*>(ctx.input(1).data());
    for (std::uint32_t i = 0; i < period; ++i) {
      gpu->host[2 * i] = re[i];
      gpu->host[2 * i + 1] = im[i];
    }
    ck(df_memcpy_h2d(gpu->ctrl, &gpu->token, 4, gpu->stream));
    ck(df_memcpy_h2d(gpu->in, gpu->host.data(), 8ull * period, gpu->stream));
    ck(df_dpd_fire(gpu->d, static_cast<const std::uint32_t*>(gpu->ctrl), static_cast<const float*>(gpu->in),
                   static_cast<float*>(gpu->out), 1, gpu->stream));
    ck(df_memcpy_d2h(gpu->host.data(), gpu->out, 8ull * period, gpu->stream));
    ck(df_stream_synchronize(gpu->stream));
    float* ore = reinterpret_cast<float*>(ctx.output(0).data());
    float* oim = reinterpret_cast<float*>(ctx.output(1).data());
    for (std::uint32_t i = 0; i < period; ++i) {
      ore[i] = gpu->host[2 * i];
      oim[i] = gpu->host[2 * i + 1];
    }
  };
  dpd_gpu.finish = [gpu] { ck(df_dpd_error(gpu->d)); };
  const auto out = std::span<std::complex<float>>(output);
  ActorBehavior sink;  // dpd.cpp:333-347
  sink.fire = [out, period](FiringContext& ctx) {
    const float* re = reinterpret_cast<const float*>(ctx.input(0).data());
    const float* im = reinterpret_cast<const float*>(ctx.input(1).data());
    const std::size_t base = ctx.firing_index() * period;
    for (std::size_t i = 0; i < period; ++i) out[base + i] = {re[i], im[i]};
  };
  using PD = PortDirection;
  using PK = PortKind;
  std::vector<ActorSpec> actors = {
      {"source", ActorKind::static_rate, {{PD::output, PK::regular, "src_re"}, {PD::output, PK::regular, "src_im"}}, source, {}},
      {"config", ActorKind::static_rate, {{PD::output, PK::regular, "cfg_gpu"}}, config, {}},
      {"dpd_gpu",
       ActorKind::dynamic_rate,
       {{PD::input, PK::control, "cfg_gpu"},
        {PD::input, PK::regular, "src_re"},
        {PD::input, PK::regular, "src_im"},
        {PD::output, PK::regular, "gpu_re"},
        {PD::output, PK::regular, "gpu_im"}},
       dpd_gpu,
       {}},
      {"sink", ActorKind::static_rate, {{PD::input, PK::regular, "gpu_re"}, {PD::input, PK::regular, "gpu_im"}}, sink, {}},
  };
  ExecutionConfig cfg;
  cfg.source_firing_limit = p.samples / period;
  run(build_network(actors, channels), cfg);
  return output;
}

bool same_bits(const std::vector<std::complex<float>>& a, const std::vector<std::complex<float>>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(a[0])) == 0;
}

}  // namespace

int main() {
  try {
    const unsigned w = 320, h = 240;
    const auto frames = motion::synth_frames(64, w, h, 606);  // acceptance.cpp:328-341
    const auto want = motion::oracle_motion_detection_raw(frames, w, h, 32);
    for (std::uint32_t r : {1u, 4u}) {
      const auto got = run_motion_dropin(frames, w, h, 32, r);
      report("motion_r" + std::to_string(r), got == want);
    }
  } catch (const std::exception& e) {
    report("motion", false, e.what());
  }
  try {
    dpd::Params p;  // acceptance.cpp:376-395
    p.period = 65536;
    p.samples = 1ull << 20;
    p.taps = dpd::random_taps(808);
    p.schedule = dpd::random_schedule(16, 809);
    const auto input = dpd::synth_samples(p.samples, 810);
    p.input = input;
    const auto got = run_dpd_dropin(p);
    report("dpd_acc8", same_bits(got, dpd::oracle_dpd(input, p.taps, p.schedule, p.period)));
    p.period = 4096;
    p.samples = 4096ull * 64;
    p.schedule = dpd::random_schedule(23, 2020);
    const auto input2 = dpd::synth_samples(p.samples, 2021);
    p.input = input2;
    const auto got2 = run_dpd_dropin(p);
    report("dpd_p4096", same_bits(got2, dpd::oracle_dpd(input2, p.taps, p.schedule, p.period)));
  } catch (const std::exception& e) {
    report("dpd", false, e.what());
  }
  try {  // the GPU actor's C-ABI call fails (null output buffer) inside fire
    const auto frames = motion::synth_frames(4, 64, 48, 1);
    run_motion_dropin(frames, 64, 48, 32, 1, true);
    report("fault", false, "run() returned");
  } catch (const ActorFault& e) {
    report("fault", std::string(e.what()).find("motion_gpu") != std::string::npos, e.what());
  } catch (const std::exception& e) {
    report("fault", false, std::string("wrong exception: ") + e.what());
  }
  return failures ? 1 : 0;
}
