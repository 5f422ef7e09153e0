// Tuning knobs: explicit, process-wide overrides of the engine's planning and
// launch choices (loop width, pairing mode, banded tables, autotuning, ...).
//
// They exist for the tests (which force every kernel variant against the
// oracle) and for the experiment scripts under tools/.  They are set only
// through isd_set_knob(); the library never reads the environment, so a
// caller's environment cannot change plans, kernels or timings.  Every knob
// that is set enters the plan-cache key (knob_signature), so plans made
// under one knob set are never reused under another.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "isd_internal.h"

namespace isd {

namespace {
std::mutex g_knob_mu;
std::map<std::string, std::string> g_knobs;

// every knob the library consults (a typo is an error, not a silent no-op)
const char* const kKnownKnobs[] = {
    "ISD_AUTOTUNE",          "ISD_BAND",
    "ISD_BAND_CALIBRATE",
    "ISD_BAND_DOMINO",       "ISD_BAND_DOMINO_LOOP_BITS",
    "ISD_BAND_DYNAMIC",      "ISD_BAND_ITEMS_PER_SM",
    "ISD_BAND_LOOP_BITS",    "ISD_BAND_MIRROR",
    "ISD_BAND_ORDER",        "ISD_BAND_SPAN",
    "ISD_BAND_WEIGHTS",      "ISD_CLIMB_STARTS",
    "ISD_CLIMB_STEPS",       "ISD_COPY_VARIANT",
    "ISD_GPU_CLIMB",         "ISD_GRAY",
    "ISD_GRID_SMS",          "ISD_HIST_BYTES",
    "ISD_JIT",               "ISD_JIT_DUMP",
    "ISD_LAYOUT",            "ISD_LOOP_BITS",
    "ISD_NHIST_MAX",         "ISD_PAIR",
    "ISD_PEER",
    "ISD_PLAN_TOP",          "ISD_PLAN_WIDE",
    "ISD_PROBE",             "ISD_TUNE_CANDIDATES",
    "ISD_TUNE_FINALISTS",    "ISD_TUNE_BANDED",
};
}  // namespace

bool knob_known(const char* name) {
  for (const char* k : kKnownKnobs)
    if (std::strcmp(k, name) == 0) return true;
  return false;
}

bool knob_str(const char* name, std::string* out) {
  std::lock_guard<std::mutex> lock(g_knob_mu);
  auto it = g_knobs.find(name);
  if (it == g_knobs.end()) return false;
  if (out) *out = it->second;
  return true;
}

long knob_long(const char* name, long dflt) {
  std::string v;
  if (!knob_str(name, &v) || v.empty()) return dflt;
  char* end = nullptr;
  const long x = std::strtol(v.c_str(), &end, 10);
  return (end && *end == 0) ? x : dflt;
}

std::string knob_signature() {
  std::lock_guard<std::mutex> lock(g_knob_mu);
  std::string s;
  for (const auto& kv : g_knobs) s += "|" + kv.first + "=" + kv.second;
  return s;
}

int set_knob(const char* name, const char* value) {
  std::lock_guard<std::mutex> lock(g_knob_mu);
  if (!value || !*value)
    g_knobs.erase(name);
  else
    g_knobs[name] = value;
  return ISD_OK;
}

void clear_knobs() {
  std::lock_guard<std::mutex> lock(g_knob_mu);
  g_knobs.clear();
}

}  // namespace isd
