// Tuning / A-B switches: LF_* names read where they take
// effect -- plan creation (code generation, executor choice) or launch.  An
// in-process override set by lf_set_option wins over the environment, so a
// host (or a test) can flip a switch between plans without a new process.
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>

#include "exec.hpp"

namespace lfx {

namespace {
std::mutex g_mu;
std::map<std::string, const char*> g_over;  // name -> value (nullptr: unset, environment ignored)
std::deque<std::string> g_store;            // values, never freed (returned pointers stay valid)
}  // namespace

const char* option(const char* name) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_over.find(name);
    if (it != g_over.end()) return it->second;
  }
  return std::getenv(name);
}

int set_option(const char* name, const char* value, int clear) {
  if (!name || std::strncmp(name, "LF_", 3) != 0) return -1;
  std::lock_guard<std::mutex> lk(g_mu);
  if (clear) {
    g_over.erase(name);
    return 0;
  }
  if (!value) {
    g_over[name] = nullptr;
    return 0;
  }
  g_store.emplace_back(value);
  g_over[name] = g_store.back().c_str();
  return 0;
}

}  // namespace lfx
