// sd_rworker: the reference CLI's `serve` subcommand (splitdecode_main.cpp:
// cmd_serve, ServeOptions workers.hpp:68-74) on a B200: an attention worker
// speaking SDWP over TCP with its KV shard in HBM. Options mirror the
// reference's: --listen host:port (port 0 = ephemeral), --capacity tokens
// (required), --storage single|half|int8, --port-file, --once, --timeout s;
// plus --device. Built against the C ABI only, through its C++ face
// (include/sd_b200.hpp: ServeOptions, serve_attention_worker).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/sd_b200.hpp"

static int usage() {
  std::fprintf(stderr,
               "usage: sd_rworker serve --capacity TOKENS [--listen HOST:PORT] [--storage single|half|int8|int4]\n"
               "                        [--port-file PATH] [--once] [--timeout SECONDS] [--device N]\n");
  return 2;
}

int main(int argc, char** argv) {
  if (argc < 2 || std::strcmp(argv[1], "serve") != 0) return usage();
  std::string listen = "127.0.0.1:0", storage = "single", port_file;
  long long capacity = -1;
  int once = 0, device = 0;
  double timeout = 0;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> const char* {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "sd_rworker: %s needs a value\n", a.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (a == "--listen") {
      listen = val();
    } else if (a == "--capacity") {
      capacity = std::atoll(val());
    } else if (a == "--storage") {
      storage = val();
    } else if (a == "--port-file") {
      port_file = val();
    } else if (a == "--once") {
      once = 1;
    } else if (a == "--timeout") {
      timeout = std::atof(val());
    } else if (a == "--device") {
      device = std::atoi(val());
    } else {
      return usage();
    }
  }
  if (capacity < 1) return usage();
  sd_b200::ServeOptions opts;
  opts.listen_addr = listen;
  opts.port_file = port_file;
  opts.once = once != 0;
  opts.recv_timeout_seconds = timeout;
  opts.worker.capacity_tokens = static_cast<long>(capacity);
  opts.worker.device = device;
  if (storage == "single") {
    opts.worker.storage = sd_b200::KvFormat::kSingle;
  } else if (storage == "half") {
    opts.worker.storage = sd_b200::KvFormat::kHalf;
  } else if (storage == "int8") {
    opts.worker.storage = sd_b200::KvFormat::kInt8;
  } else if (storage == "int4") {  // extension (sd_abi.h)
    opts.worker.storage = sd_b200::KvFormat::kInt4;
  } else {
    std::fprintf(stderr, "sd_rworker: unknown kv storage format: %s\n", storage.c_str());
    return 2;
  }
  try {
    sd_b200::serve_attention_worker(opts);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "sd_rworker: %s\n", e.what());
    return 1;
  }
  return 0;
}
