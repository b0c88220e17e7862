// TEST HARNESS ONLY: the trace-record parser of csrc/jsonl.cuh compiled for
// the host so the CPU test suite can fuzz it line by line against the
// compiled reference (nlohmann).  Never loaded by the product path, which
// runs the same parser only on the GPU (csrc/k_ingest.cu).
#include "jsonl.cuh"

namespace {
struct JHost {
  const unsigned char* p;
  int n;
  int operator()(int i) const { return i < n ? static_cast<int>(p[i]) : -1; }
};
}  // namespace

// out: status, reason, text, n_img, n_aud, fast; vals: image then audio values
extern "C" int jh_parse(const char* b, int len, long long cap, long long* out, int* vals,
                        int cap_vals) {
  const JHost at{reinterpret_cast<const unsigned char*>(b), len};
  bool fast = false;
  const dtb::JLine r = dtb::j_parse_record(at, len, cap, &fast);
  out[0] = r.status;
  out[1] = r.reason;
  out[2] = r.text;
  out[3] = r.n_img;
  out[4] = r.n_aud;
  out[5] = fast ? 1 : 0;
  if (r.status == dtb::J_OK && r.n_img + r.n_aud <= cap_vals) {
    if (fast) {
      if (r.img_at >= 0) dtb::j_write_array_fast(at, r.img_at, vals);
      if (r.aud_at >= 0) dtb::j_write_array_fast(at, r.aud_at, vals + r.n_img);
    } else {
      if (r.img_at >= 0) dtb::j_write_array(at, r.img_at, vals);
      if (r.aud_at >= 0) dtb::j_write_array(at, r.aud_at, vals + r.n_img);
    }
  }
  return r.status;
}

// number conversion alone: returns 1 on overflow
extern "C" int jh_number(const char* b, int len, long long* out) {
  const JHost at{reinterpret_cast<const unsigned char*>(b), len};
  const int e = dtb::j_number_end(at, 0);
  if (e != len) return -1;
  return dtb::j_number_value(at, 0, e, out);
}
