// On-disk cache of the engine's expensive per-lattice artefacts: autotuned
// plans, band cost curves and NVRTC cubins ("cold start").
//
// A cold c5 walk otherwise spends seconds before its first kernel: the
// layout model (~3 s of host CPU), the GPU autotune of the model's best
// layouts, and one NVRTC compile per finalist.  With the cache a new process
// loads the tuned plan, the cost curve and the cubin instead, so the plan a
// lattice runs with is also the same in every process.
//
// Layout: a list of directories (isd_set_cache_dirs); the first is written,
// the others are read-only seeds.  One file per entry, named by a 128-bit
// hash of its key; the file stores the full key, so a hash collision is a
// miss, never a wrong plan, and a checksum of the payload, so a torn or
// corrupted file is a miss too.  Writes go to a temporary file and are renamed
// into place (atomic for concurrent processes).  Keys carry ISD_BUILD_ID (a
// hash of the library sources, set by _build.py), so a rebuilt library never
// reads another build's entries.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <sys/stat.h>
#include <unistd.h>

#include "isd_internal.h"

#ifndef ISD_BUILD_ID
#define ISD_BUILD_ID "unversioned"
#endif

namespace isd {

namespace {
std::mutex g_cache_mu;
std::vector<std::string> g_dirs;  // [0] is written, the rest are read-only
std::atomic<unsigned> g_tmp_seq{0};

constexpr char kMagic[8] = {'I', 'S', 'D', 'C', 'A', 'C', 'H', '2'};

uint64_t fnv1a(const std::string& s, uint64_t h) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::string file_name(const std::string& kind, const std::string& key) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%016llx%016llx",
                (unsigned long long)fnv1a(key, 1469598103934665603ull),
                (unsigned long long)fnv1a(key, 0x9E3779B97F4A7C15ull));
  return kind + "-" + buf + ".bin";
}

bool read_file(const std::string& path, std::string* data) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  std::string d;
  char buf[65536];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) d.append(buf, n);
  std::fclose(f);
  *data = std::move(d);
  return true;
}
}  // namespace

const char* build_id() { return ISD_BUILD_ID; }

void set_cache_dirs(const std::string& list) {
  std::vector<std::string> dirs;
  size_t a = 0;
  while (a <= list.size()) {
    size_t b = list.find(':', a);
    if (b == std::string::npos) b = list.size();
    if (b > a) dirs.push_back(list.substr(a, b - a));
    a = b + 1;
  }
  std::lock_guard<std::mutex> lock(g_cache_mu);
  g_dirs = std::move(dirs);
}

std::string cache_dirs() {
  std::lock_guard<std::mutex> lock(g_cache_mu);
  std::string s;
  for (size_t i = 0; i < g_dirs.size(); ++i) s += (i ? ":" : "") + g_dirs[i];
  return s;
}

bool cache_get(const std::string& kind, const std::string& key,
               std::string* blob) {
  std::vector<std::string> dirs;
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    dirs = g_dirs;
  }
  const std::string full = std::string(ISD_BUILD_ID) + "|" + key;
  const std::string name = file_name(kind, full);
  for (const std::string& d : dirs) {
    std::string data;
    if (!read_file(d + "/" + name, &data)) continue;
    // magic | u64 key length | key | u64 FNV-1a of the blob | blob
    if (data.size() < 24 || std::memcmp(data.data(), kMagic, 8) != 0)
      continue;
    uint64_t klen = 0, sum = 0;
    std::memcpy(&klen, data.data() + 8, 8);
    if (data.size() < 24 + klen || data.compare(16, klen, full) != 0) continue;
    std::memcpy(&sum, data.data() + 16 + klen, 8);
    std::string b = data.substr(24 + klen);
    if (fnv1a(b, 1469598103934665603ull) != sum) continue;  // torn / corrupt
    *blob = std::move(b);
    return true;
  }
  return false;
}

void cache_put(const std::string& kind, const std::string& key,
               const std::string& blob) {
  std::string dir;
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    if (g_dirs.empty()) return;
    dir = g_dirs[0];
  }
  // create the directory and its parents
  for (size_t i = 1; i <= dir.size(); ++i)
    if (i == dir.size() || dir[i] == '/') ::mkdir(dir.substr(0, i).c_str(), 0755);
  const std::string full = std::string(ISD_BUILD_ID) + "|" + key;
  const std::string path = dir + "/" + file_name(kind, full);
  const std::string tmp =
      path + ".tmp" + std::to_string((long long)::getpid()) + "." +
      std::to_string(g_tmp_seq.fetch_add(1));
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;  // a read-only or missing cache is not an error
  const uint64_t klen = full.size();
  const uint64_t sum = fnv1a(blob, 1469598103934665603ull);
  bool ok = std::fwrite(kMagic, 1, 8, f) == 8 &&
            std::fwrite(&klen, 1, 8, f) == 8 &&
            std::fwrite(full.data(), 1, full.size(), f) == full.size() &&
            std::fwrite(&sum, 1, 8, f) == 8 &&
            std::fwrite(blob.data(), 1, blob.size(), f) == blob.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0)
    std::remove(tmp.c_str());
}

}  // namespace isd
