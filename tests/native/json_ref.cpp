// TEST HARNESS ONLY: nlohmann::json 3.11.3 (the reference's JSON library,
// SURVEY.md §8(c)) applied to one number token the way ingest_trace applies
// it (json::parse + get<int64_t>, src/workload.cpp:125-134).
#include <cstdint>
#include <string>

#include <nlohmann/json.hpp>

// returns 0 ok (*out = value), 1 parse error (incl. overflow), 2 type error
extern "C" int jref_number(const char* b, int len, long long* out) {
  try {
    const auto j = nlohmann::json::parse(std::string(b, static_cast<size_t>(len)));
    try {
      *out = j.get<std::int64_t>();
      return 0;
    } catch (const std::exception&) {
      return 2;
    }
  } catch (const std::exception&) {
    return 1;
  }
}
