// mmx_tune -- command-line front end of the host layer: the reference's `acctune analyze | tune | report`
// (/root/reference/proj/tools/acctune.cpp:9-47) over the CUDA / sim backends of this build.
//
//   mmx_tune analyze <config.json>
//   mmx_tune tune    <config.json> [--seed N] [--sim model.json]
//   mmx_tune report  <workdir>
//   mmx_tune calibrate <config.json>      (cuda backend: measured times -> calibrated_model.json)
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <string>

#include "mmxhost/commands.hpp"

namespace {

int usage() {
  std::cerr << "usage: mmx_tune analyze <config.json>\n"
               "       mmx_tune tune <config.json> [--seed N] [--sim model.json]\n"
               "       mmx_tune report <workdir>\n"
               "       mmx_tune calibrate <config.json>\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  const std::string cmd = argv[1], target = argv[2];
  if (cmd == "analyze" && argc == 3) return mmxhost::cmd_analyze(target, std::cout, std::cerr);
  if (cmd == "report" && argc == 3) return mmxhost::cmd_report(target, std::cout, std::cerr);
  if (cmd == "calibrate" && argc == 3) return mmxhost::cmd_calibrate(target, std::cout, std::cerr);
  if (cmd == "tune") {
    mmxhost::TuneOptions opt;
    for (int i = 3; i < argc; ++i) {
      const std::string a = argv[i];
      if (a == "--seed" && i + 1 < argc) {
        char* end = nullptr;
        const unsigned long long v = std::strtoull(argv[++i], &end, 10);
        if (end == nullptr || *end != '\0') return usage();
        opt.seed = static_cast<std::uint64_t>(v);
      } else if (a == "--sim" && i + 1 < argc) {
        opt.sim_model = argv[++i];
      } else {
        return usage();
      }
    }
    return mmxhost::cmd_tune(target, opt, std::cout, std::cerr);
  }
  return usage();
}
