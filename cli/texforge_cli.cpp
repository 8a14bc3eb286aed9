// texforge — command-line front end of the B200 GLCM engine.
//
// Same subcommands, flags, output files and exit codes as the reference CLI
// (R/tools/texforge.cpp: compute | synth | features | bench; exit codes
// 0 ok / 1 usage / 2 input / 3 computation, :21-24), written over the drop-in
// headers in include/texforge/, so every scheme runs on the GPU. One more
// scheme, `device`, names the engine's direct path (the fused vote kernel;
// equal to `serial` on the drop-in, kept so scripts can ask for it
// explicitly). Argument parsing is a small hand-written parser (the
// reference uses CLI11, absent from this image); JSON goes out through a
// minimal ordered emitter.
#include <cstdio>
#include <fstream>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "texforge/texforge.hpp"

namespace {

constexpr int kOk = 0, kUsage = 1, kInput = 2, kCompute = 3;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- arguments -------------------------------------------------------------
class Args {
 public:
  Args(int argc, char** argv, const std::set<std::string>& flags) {
    for (int i = 2; i < argc; ++i) {
      std::string k = argv[i];
      if (k.rfind("--", 0) != 0) throw UsageError("unexpected argument " + k);
      std::string v;
      const auto eq = k.find('=');
      if (eq != std::string::npos) {
        v = k.substr(eq + 1);
        k = k.substr(0, eq);
      } else if (flags.count(k)) {
        v = "1";
      } else {
        if (i + 1 >= argc) throw UsageError(k + " needs a value");
        v = argv[++i];
      }
      kv_[k] = v;
    }
  }
  bool has(const std::string& k) const { return kv_.count(k) != 0; }
  std::string str(const std::string& k, std::optional<std::string> def = std::nullopt) {
    used_.insert(k);
    if (!has(k)) {
      if (!def) throw UsageError(k + " is required");
      return *def;
    }
    return kv_.at(k);
  }
  long num(const std::string& k, std::optional<long> def, long lo, long hi) {
    used_.insert(k);
    if (!has(k)) {
      if (!def) throw UsageError(k + " is required");
      return *def;
    }
    char* end = nullptr;
    const long v = std::strtol(kv_.at(k).c_str(), &end, 10);
    if (!end || *end || v < lo || v > hi) throw UsageError(k + " out of range");
    return v;
  }
  std::vector<std::string> list(const std::string& k, const std::vector<std::string>& def) {
    used_.insert(k);
    if (!has(k)) return def;
    std::vector<std::string> out;
    std::stringstream ss(kv_.at(k));
    for (std::string item; std::getline(ss, item, ',');)
      if (!item.empty()) out.push_back(item);
    if (out.empty()) throw UsageError(k + " is empty");
    return out;
  }
  bool flag(const std::string& k) {
    used_.insert(k);
    return has(k);
  }
  void done() const {
    for (const auto& [k, v] : kv_)
      if (!used_.count(k)) throw UsageError("unknown option " + k);
  }

 private:
  std::map<std::string, std::string> kv_;
  std::set<std::string> used_;
};

std::string member(const std::string& v, const std::set<std::string>& allowed, const char* what) {
  if (!allowed.count(v)) throw UsageError(std::string(what) + " must be one of the listed values");
  return v;
}

int angle_arg(Args& a, std::optional<long> def) {
  const long v = a.num("--angle", def, 0, 135);
  if (v != 0 && v != 45 && v != 90 && v != 135) throw UsageError("--angle must be 0, 45, 90 or 135");
  return static_cast<int>(v);
}

const std::set<std::string> kSchemes = {"serial", "shared", "privatized", "pipelined", "device"};

// ---- JSON (ordered, minimal) -------------------------------------------------
class Json {
 public:
  Json& kv(const std::string& k, const std::string& raw) {
    body_ += (body_.empty() ? "" : ",") + ("\"" + k + "\":" + raw);
    return *this;
  }
  Json& num(const std::string& k, double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return kv(k, b);
  }
  Json& num(const std::string& k, unsigned long long v) { return kv(k, std::to_string(v)); }
  Json& num(const std::string& k, long long v) { return kv(k, std::to_string(v)); }
  Json& num(const std::string& k, int v) { return kv(k, std::to_string(v)); }
  Json& boolean(const std::string& k, bool v) { return kv(k, v ? "true" : "false"); }
  Json& text(const std::string& k, const std::string& v) { return kv(k, "\"" + v + "\""); }
  std::string dump() const { return "{" + body_ + "}"; }

 private:
  std::string body_;
};

std::string contention_json(const texforge::ContentionStats& s) {
  Json j;
  j.num("total_votes", (unsigned long long)s.total_votes)
      .num("hottest_cell_votes", (unsigned long long)s.hottest_cell_votes)
      .kv("hottest_cell",
          "[" + std::to_string(s.hottest_cell_index.first) + "," + std::to_string(s.hottest_cell_index.second) + "]")
      .num("concentration", s.concentration);
  if (!s.per_copy_hottest.empty()) {
    std::string arr = "[";
    for (std::size_t i = 0; i < s.per_copy_hottest.size(); ++i)
      arr += (i ? "," : "") + std::to_string(s.per_copy_hottest[i]);
    j.kv("per_copy_hottest", arr + "]");
  }
  return j.dump();
}

// ---- schemes -----------------------------------------------------------------
std::size_t auto_chunks(std::size_t height, int distance) {
  const std::size_t cap = height / (static_cast<std::size_t>(distance) + 1);
  return std::max<std::size_t>(1, std::min<std::size_t>(8, cap));
}

struct Run {
  texforge::Glcm glcm;
  std::optional<texforge::ContentionStats> contention;
};

Run run_scheme(const std::string& scheme, const std::string& path, const texforge::GlcmParams& p, unsigned copies,
               std::size_t chunks) {
  texforge::ExecutionPlan plan = texforge::plan(p.levels, texforge::kDefaultScratchBudget, texforge::detect_worker_count());
  if (copies) plan.copies = copies;
  if (scheme == "pipelined") {
    texforge::PgmChunkSource src(path, p.levels);
    return {texforge::compute_glcm_chunked(src, p, plan, chunks ? chunks : auto_chunks(src.height(), p.distance)),
            std::nullopt};
  }
  const texforge::QuantizedImage img = texforge::quantize(texforge::load_pgm_file(path), p.levels);
  if (scheme == "serial" || scheme == "device") return {texforge::compute_glcm_serial(img, p), std::nullopt};
  auto [g, st] = scheme == "shared" ? texforge::compute_glcm_shared(img, p, plan)
                                    : texforge::compute_glcm_privatized(img, p, plan);
  return {std::move(g), std::move(st)};
}

texforge::PgmHeader header_of(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw texforge::PgmError("pgm: cannot open " + path);
  std::vector<std::uint8_t> head(4096);
  in.read(reinterpret_cast<char*>(head.data()), static_cast<std::streamsize>(head.size()));
  head.resize(static_cast<std::size_t>(in.gcount()));
  return texforge::parse_pgm_header(head);
}

// ---- subcommands ---------------------------------------------------------------
int cmd_compute(Args& a) {
  const std::string input = a.str("--input"), output = a.str("--output");
  const int levels = static_cast<int>(a.num("--levels", std::nullopt, 2, 256));
  const int distance = static_cast<int>(a.num("--distance", std::nullopt, 1, 1L << 30));
  const int angle = angle_arg(a, std::nullopt);
  const std::string scheme = member(a.str("--scheme", "serial"), kSchemes, "--scheme");
  const unsigned copies = static_cast<unsigned>(a.num("--copies", 0, 0, 64));
  const std::size_t chunks = static_cast<std::size_t>(a.num("--chunks", 0, 0, 1L << 30));
  const bool symmetric = a.flag("--symmetric"), normalized = a.flag("--normalize");
  a.done();

  const texforge::GlcmParams p{distance, texforge::angle_from_degrees(angle), levels};
  const texforge::PgmHeader h = header_of(input);
  Run run = run_scheme(scheme, input, p, copies, chunks);
  std::ofstream out(output, std::ios::binary);
  if (!out) {
    std::cerr << "error: cannot create " << output << "\n";
    return kInput;
  }
  const texforge::Glcm final_glcm = symmetric ? texforge::symmetrize(run.glcm) : run.glcm;
  if (normalized)
    texforge::write_probabilities_csv(texforge::normalize(final_glcm), out);
  else
    texforge::write_glcm_csv(final_glcm, out);
  Json j;
  j.text("scheme", scheme).num("levels", levels).num("distance", distance).num("angle", angle);
  j.num("total_votes", (unsigned long long)run.glcm.total());
  j.num("valid_pair_count", (unsigned long long)texforge::valid_pair_count(h.width, h.height, p));
  j.boolean("symmetric", symmetric);
  if (run.contention) j.kv("contention", contention_json(*run.contention));
  std::cout << j.dump() << "\n";
  return kOk;
}

int cmd_synth(Args& a) {
  const std::string kind = member(a.str("--kind"), {"smooth", "noise"}, "--kind");
  const std::string size = a.str("--size"), output = a.str("--output");
  const long seed = a.num("--seed", 1, 0, 0xFFFFFFFFL);
  a.done();
  std::size_t w = 0, h = 0;
  const auto x = size.find('x');
  try {
    if (x == std::string::npos || x == 0 || x + 1 >= size.size()) throw UsageError("");
    w = std::stoull(size.substr(0, x));
    h = std::stoull(size.substr(x + 1));
  } catch (...) {
    w = h = 0;
  }
  if (w < 2 || h < 2) throw UsageError("--size must look like 512x512 (both dims >= 2)");
  const auto s = static_cast<std::uint32_t>(seed);
  texforge::write_pgm_file(kind == "smooth" ? texforge::synth_smooth(w, h, s) : texforge::synth_noise(w, h, s), output);
  return kOk;
}

int cmd_features(Args& a) {
  const std::string input = a.str("--input");
  const int levels = static_cast<int>(a.num("--levels", std::nullopt, 2, 256));
  const int distance = static_cast<int>(a.num("--distance", std::nullopt, 1, 1L << 30));
  const int angle = angle_arg(a, std::nullopt);
  const std::string scheme = member(a.str("--scheme", "serial"), kSchemes, "--scheme");
  const bool symmetric = a.flag("--symmetric");
  a.done();
  const texforge::GlcmParams p{distance, texforge::angle_from_degrees(angle), levels};
  Run run = run_scheme(scheme, input, p, 0, 0);
  const texforge::FeatureVector f =
      texforge::extract_features(texforge::normalize(symmetric ? texforge::symmetrize(run.glcm) : run.glcm));
  Json j;
  j.num("energy", f.energy).num("contrast", f.contrast).num("homogeneity", f.homogeneity);
  j.num("entropy", f.entropy).num("correlation", f.correlation);
  std::cout << j.dump() << "\n";
  return kOk;
}

int cmd_bench(Args& a) {
  std::vector<std::size_t> sizes;
  for (const auto& s : a.list("--sizes", {"1024"})) sizes.push_back(std::stoull(s));
  std::vector<int> levels_list;
  for (const auto& s : a.list("--levels", {"8", "32"})) levels_list.push_back(std::stoi(s));
  const auto images = a.list("--images", {"smooth", "noise"});
  for (const auto& i : images) member(i, {"smooth", "noise"}, "--images");
  const auto schemes = a.list("--schemes", {"serial", "shared", "privatized", "pipelined"});
  for (const auto& s : schemes) member(s, kSchemes, "--schemes");
  const int repeats = static_cast<int>(a.num("--repeats", 20, 1, 1L << 30));
  const int distance = static_cast<int>(a.num("--distance", 1, 1, 1L << 30));
  const int angle = angle_arg(a, 0);
  const std::size_t chunks_opt = static_cast<std::size_t>(a.num("--chunks", 8, 0, 1L << 30));
  const auto seed = static_cast<std::uint32_t>(a.num("--seed", 1, 0, 0xFFFFFFFFL));
  const std::string ingest = member(a.str("--ingest", "none"), {"none", "matched", "doubled"}, "--ingest");
  const std::string output = a.str("--output", "report.csv");
  a.done();

  const unsigned workers = texforge::detect_worker_count();
  std::vector<texforge::BenchRow> rows;
  for (std::size_t n : sizes) {
    for (const std::string& kind : images) {
      const texforge::GrayImage gray = kind == "smooth" ? texforge::synth_smooth(n, n, seed)
                                                        : texforge::synth_noise(n, n, seed);
      for (int L : levels_list) {
        const texforge::QuantizedImage img = texforge::quantize(gray, L);
        const texforge::GlcmParams p{distance, texforge::angle_from_degrees(angle), L};
        const texforge::ExecutionPlan plan = texforge::plan(L, texforge::kDefaultScratchBudget, workers);
        const std::size_t chunks = chunks_opt ? chunks_opt : auto_chunks(img.height, distance);
        double ns_per_byte = 0.0;  // synthetic link calibrated on this configuration (texforge.cpp:206-215)
        if (ingest != "none") {
          const double t = texforge::time_once_ms([&] { texforge::compute_glcm_privatized(img, p, plan); });
          ns_per_byte = t * 1e6 / static_cast<double>(img.pixels.size()) * (ingest == "doubled" ? 2.0 : 1.0);
        }
        double serial_mean = 0.0;
        for (const std::string& scheme : schemes) {
          auto once = [&] {
            if (scheme == "pipelined") {
              texforge::MemoryChunkSource mem(img);
              texforge::LatencyChunkSource src(mem, ns_per_byte);
              texforge::compute_glcm_chunked(src, p, plan, chunks);
              return;
            }
            texforge::detail::simulate_full_ingest(img.pixels.size(), ns_per_byte);
            if (scheme == "serial" || scheme == "device") texforge::compute_glcm_serial(img, p);
            else if (scheme == "shared") texforge::compute_glcm_shared(img, p, plan);
            else texforge::compute_glcm_privatized(img, p, plan);
          };
          texforge::BenchRow r;
          r.scheme = scheme;
          r.image = kind;
          r.width = r.height = n;
          r.levels = L;
          r.distance = distance;
          r.angle_deg = angle;
          r.copies = (scheme == "privatized" || scheme == "pipelined") ? plan.copies : 0;
          r.chunks = scheme == "pipelined" ? chunks : 0;
          r.timing = texforge::summarize_ms(texforge::time_repeats_ms(repeats, once));
          if (scheme == "serial") serial_mean = r.timing.mean_ms;
          r.speedup_vs_serial = serial_mean > 0.0 ? serial_mean / r.timing.mean_ms : 1.0;
          rows.push_back(r);
          std::printf("%zux%zu %s L=%-3d %-10s mean %8.3f ms  std %7.3f  median %8.3f  speedup %.2fx\n", n, n,
                      kind.c_str(), L, scheme.c_str(), r.timing.mean_ms, r.timing.std_ms, r.timing.median_ms,
                      r.speedup_vs_serial);
        }
      }
    }
  }
  std::ofstream out(output, std::ios::binary);
  if (!out) {
    std::cerr << "error: cannot create " << output << "\n";
    return kInput;
  }
  texforge::write_bench_csv(rows, out);
  std::printf("report written to %s (%zu rows, %u workers)\n", output.c_str(), rows.size(), workers);
  return kOk;
}

const char* kUsageText =
    "usage: texforge <compute|synth|features|bench> [options]\n"
    "  compute  --input PGM --output CSV --levels L --distance D --angle A\n"
    "           [--scheme serial|shared|privatized|pipelined|device] [--copies R] [--chunks K]\n"
    "           [--symmetric] [--normalize]\n"
    "  synth    --kind smooth|noise --size WxH --output PGM [--seed S]\n"
    "  features --input PGM --levels L --distance D --angle A [--scheme ...] [--symmetric]\n"
    "  bench    [--sizes N,..] [--levels L,..] [--images smooth,noise] [--schemes ...]\n"
    "           [--repeats N] [--distance D] [--angle A] [--chunks K] [--seed S]\n"
    "           [--ingest none|matched|doubled] [--output CSV]\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsageText;
    return kUsage;
  }
  const std::string cmd = argv[1];
  const std::map<std::string, std::pair<std::set<std::string>, std::function<int(Args&)>>> table = {
      {"compute", {{"--symmetric", "--normalize"}, cmd_compute}},
      {"synth", {{}, cmd_synth}},
      {"features", {{"--symmetric"}, cmd_features}},
      {"bench", {{}, cmd_bench}},
  };
  const auto it = table.find(cmd);
  if (it == table.end()) {
    std::cerr << kUsageText;
    return (cmd == "--help" || cmd == "-h") ? kOk : kUsage;
  }
  try {
    Args args(argc, argv, it->second.first);
    return it->second.second(args);
  } catch (const UsageError& e) {
    std::cerr << "usage error: " << e.what() << "\n" << kUsageText;
    return kUsage;
  } catch (const texforge::PgmError& e) {
    std::cerr << "input error: " << e.what() << "\n";
    return kInput;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kCompute;
  }
}
