// The reference's "distributed generation equals the monolithic oracle"
// cases (proj/tests/test_workers.cpp:280-332) restated against the C++
// interface of include/sd_b200.hpp: one forked process per rank, all on one
// device, the peer exchange connected through pipes to the parent (which
// gathers the CUDA IPC handles in rank order); each rank drives the
// schedule and reports its home rows, and the union must equal the
// monolithic transcript row for row. The parent touches CUDA only after
// every child has exited (a forked child cannot inherit a CUDA context).
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "sd_b200.hpp"

using namespace sd_b200;

namespace {

struct Case {
  const char* name;
  int world, s_ranks;
  ShardMode mode;
  bool pipelined;
  GenerationConfig cfg;
};

GenerationConfig toy_config(int batch, int target_len, int interval, long steps) {  // test_workers.cpp:23-34
  GenerationConfig c;
  c.seed = 0;
  c.batch = batch;
  c.target_len = target_len;
  c.interval = interval;
  c.steps = steps;
  return c;
}

bool write_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t k = write(fd, c, n);
    if (k <= 0) return false;
    c += k;
    n -= static_cast<size_t>(k);
  }
  return true;
}
bool read_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t k = read(fd, c, n);
    if (k <= 0) return false;
    c += k;
    n -= static_cast<size_t>(k);
  }
  return true;
}

// one rank: build its shard and computation, exchange IPC handles through
// the parent, drive the schedule, send back its rows
int run_rank(const Case& c, int rank, int up, int down) {
  try {
    const ModelSpec spec = make_model_spec(2, 64, 4, 256, 128);  // kToySpec
    const bool is_s = c.s_ranks == c.world || rank == 0;
    std::unique_ptr<WeightSet> w;
    if (is_s) w = std::make_unique<WeightSet>(spec, c.cfg.seed);
    const auto [h0, hc] = c.mode == ShardMode::kBySequence ? std::pair<int, int>{0, spec.num_heads}
                                                           : shard_head_range(c.mode, spec.num_heads, c.world, rank);
    KvShard kv(spec, h0, hc, 1 << 16);
    DistributedComputation dist(w.get(), kv, rank, c.world, c.s_ranks, c.mode);
    const std::vector<std::uint8_t> mine = dist.setup(c.cfg.batch);
    std::vector<std::uint8_t> all(static_cast<size_t>(c.world) * SD_DIST_IPC_BYTES);
    if (!write_all(up, mine.data(), mine.size()) || !read_all(down, all.data(), all.size())) return 3;
    dist.connect(all);
    dist.set_pipelined(c.pipelined);
    const std::vector<GenerationRecord> rows = drive_schedule(c.cfg, dist);
    const std::int64_t left = kv.token_count();  // checked against the monolithic store
    const std::int64_t n = static_cast<std::int64_t>(rows.size());
    if (!write_all(up, &left, sizeof left) || !write_all(up, &n, sizeof n)) return 3;
    for (const GenerationRecord& r : rows) {
      const std::int64_t v[3] = {r.step, static_cast<std::int64_t>(r.seq), r.token};
      if (!write_all(up, v, sizeof v)) return 3;
    }
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rank %d: %s\n", rank, e.what());
    return 2;
  }
}

using Row = std::tuple<long, SequenceId, int>;

// fork the ranks, relay the handles, collect the rows and the tokens each
// shard still holds; "" on success
std::string run_distributed(const Case& c, std::vector<Row>& rows, std::vector<std::int64_t>& held) {
  std::vector<int> ups(static_cast<size_t>(c.world)), downs(static_cast<size_t>(c.world));
  std::vector<pid_t> pids;
  for (int r = 0; r < c.world; ++r) {
    int u[2], d[2];
    if (pipe(u) || pipe(d)) return "pipe failed";
    const pid_t pid = fork();
    if (pid == 0) {
      close(u[0]);
      close(d[1]);
      _exit(run_rank(c, r, u[1], d[0]));
    }
    close(u[1]);
    close(d[0]);
    ups[static_cast<size_t>(r)] = u[0];
    downs[static_cast<size_t>(r)] = d[1];
    pids.push_back(pid);
  }
  std::string err;
  std::vector<std::uint8_t> all(static_cast<size_t>(c.world) * SD_DIST_IPC_BYTES);
  for (int r = 0; r < c.world && err.empty(); ++r) {
    if (!read_all(ups[static_cast<size_t>(r)], all.data() + static_cast<size_t>(r) * SD_DIST_IPC_BYTES,
                  SD_DIST_IPC_BYTES)) {
      err = "rank " + std::to_string(r) + " sent no handles";
    }
  }
  for (int r = 0; r < c.world && err.empty(); ++r) write_all(downs[static_cast<size_t>(r)], all.data(), all.size());
  for (int r = 0; r < c.world && err.empty(); ++r) {
    std::int64_t left = 0, n = 0;
    if (!read_all(ups[static_cast<size_t>(r)], &left, sizeof left) || !read_all(ups[static_cast<size_t>(r)], &n, sizeof n)) {
      err = "rank " + std::to_string(r) + " sent no rows";
      break;
    }
    held.push_back(left);
    for (std::int64_t i = 0; i < n; ++i) {
      std::int64_t v[3];
      if (!read_all(ups[static_cast<size_t>(r)], v, sizeof v)) {
        err = "short row stream";
        break;
      }
      rows.emplace_back(static_cast<long>(v[0]), static_cast<SequenceId>(v[1]), static_cast<int>(v[2]));
    }
  }
  for (int fd : ups) close(fd);
  for (int fd : downs) close(fd);
  for (pid_t pid : pids) {
    int st = 0;
    waitpid(pid, &st, 0);
    if (err.empty() && !(WIFEXITED(st) && WEXITSTATUS(st) == 0)) err = "a rank failed";
  }
  return err;
}

}  // namespace

int main() {
  const std::vector<Case> cases = {
      {"two workers sharded by sequence", 2, 2, ShardMode::kBySequence, false, toy_config(8, 32, 32, 32)},
      {"two workers, one S-rank (the paper's topology)", 2, 1, ShardMode::kBySequence, false, toy_config(8, 32, 32, 32)},
      {"two workers sharded by head", 2, 1, ShardMode::kByHead, false, toy_config(8, 32, 32, 32)},
      {"four workers hybrid", 4, 4, ShardMode::kHybrid, false, toy_config(8, 32, 32, 32)},
      {"two interleaved mini-batches", 2, 2, ShardMode::kBySequence, true, toy_config(8, 32, 32, 32)},
      {"stabilized schedule with retirement", 2, 2, ShardMode::kBySequence, false, toy_config(8, 16, 4, 48)},
  };
  // every distributed run first: the parent initialises CUDA only afterwards
  std::vector<std::vector<Row>> got(cases.size());
  std::vector<std::vector<std::int64_t>> held(cases.size());
  std::vector<std::string> errs(cases.size());
  for (size_t i = 0; i < cases.size(); ++i) errs[i] = run_distributed(cases[i], got[i], held[i]);
  int failed = 0;
  try {
    const ModelSpec spec = make_model_spec(2, 64, 4, 256, 128);
    WeightSet w(spec, 0);
    for (size_t i = 0; i < cases.size(); ++i) {
      KvShard kv(spec, 0, spec.num_heads, 1 << 16);
      StepComputation mono(w, kv);
      std::vector<Row> want;
      for (const GenerationRecord& r : drive_schedule(cases[i].cfg, mono)) want.emplace_back(r.step, r.seq, r.token);
      std::sort(want.begin(), want.end());
      std::sort(got[i].begin(), got[i].end());
      // retirement (DROP_SEQ to every holder, workers.cpp:482-501): the
      // sequence shards together hold exactly the monolithic store's live
      // tokens; a head shard holds them all, every head shard
      const std::int64_t live = kv.token_count();
      bool drained = true;
      std::int64_t sum = 0;
      for (std::int64_t t : held[i]) {
        sum += t;
        if (cases[i].mode != ShardMode::kBySequence && live == 0) drained = drained && t == 0;
      }
      if (cases[i].mode == ShardMode::kBySequence) drained = sum == live;
      if (errs[i].empty() && !drained) errs[i] = "shards hold " + std::to_string(sum) + " tokens, expected " + std::to_string(live);
      const bool ok = errs[i].empty() && got[i] == want;
      std::printf("%s %s: %zu rows%s%s\n", ok ? "ok  " : "FAIL", cases[i].name, got[i].size(),
                  errs[i].empty() ? "" : " - ", errs[i].c_str());
      failed += ok ? 0 : 1;
    }
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught: %s\n", e.what());
    return 1;
  }
  std::printf("dist: %zu cases, %d failed\n", cases.size(), failed);
  return failed == 0 ? 0 : 1;
}
