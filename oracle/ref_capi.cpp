// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference hot path, compiled straight from
// /root/reference/proj/core/src/{eval,tables,tables_data}.cpp by oracle/Makefile
// into oracle/_ref/libboysfn_ref.so (git-ignored; it travels to the GPU box
// with the snapshot).  The reference namespace is renamed to boysfn_ref with
// -Dboysfn=boysfn_ref so it can never collide with the product's boysfn::.
// Used to pin the C restatement (oracle/boys_port.c), to generate the golden
// vectors (oracle/make_golden.py) and as bench.py's `--impl reference` arm.
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "boysfn/eval.hpp"
#include "boysfn/tables.hpp"

namespace {

// Status codes shared with oracle/boys_oracle.h and include/boysfn_b200.h.
constexpr int kOk = 0, kSize = 1, kDomain = 2, kRange = 3, kTables = 4, kParse = 8, kOther = 9;

void copy_msg(const char* what, char* msg, size_t len) {
  if (!msg || len == 0) return;
  std::strncpy(msg, what, len - 1);
  msg[len - 1] = '\0';
}

// Maps the exception types of eval.cpp:14-17,90-91 to status codes.
template <class F>
int guarded(F&& f, char* msg, size_t len) {
  try {
    f();
    return kOk;
  } catch (const boysfn::TableParseError& e) {
    copy_msg(e.what(), msg, len);
    return kParse;
  } catch (const std::domain_error& e) {
    copy_msg(e.what(), msg, len);
    return kDomain;
  } catch (const std::out_of_range& e) {
    copy_msg(e.what(), msg, len);
    return kRange;
  } catch (const std::invalid_argument& e) {
    copy_msg(e.what(), msg, len);
    return std::string(e.what()).rfind("tables:", 0) == 0 ? kTables : kSize;
  } catch (const std::exception& e) {
    copy_msg(e.what(), msg, len);
    return kOther;
  }
}

}  // namespace

extern "C" {

// boysfn::boys_batch_many (eval.hpp:44-45) on the embedded set, AoS output.
int ref_boys_batch_many(const double* xs, size_t n, int k, double* out, size_t out_len,
                        char* msg, size_t msg_len) {
  return guarded(
      [&] {
        boysfn::boys_batch_many(std::span<const double>(xs, n), k, boysfn::embedded_default(),
                                std::span<double>(out, out_len));
      },
      msg, msg_len);
}

// Same call on disjoint contiguous spans, one std::thread each (the path is
// reentrant) -- the CPU baseline of bench.py.
int ref_boys_batch_many_mt(const double* xs, size_t n, int k, double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  const auto& tables = boysfn::embedded_default();
  std::vector<std::thread> pool;
  std::vector<int> status(nthreads, kOk);
  const size_t row = static_cast<size_t>(k) + 1;
  size_t begin = 0;
  for (int w = 0; w < nthreads; ++w) {
    const size_t cnt = n / nthreads + (static_cast<size_t>(w) < n % nthreads ? 1 : 0);
    pool.emplace_back([&, w, begin, cnt] {
      status[w] = guarded(
          [&] {
            boysfn::boys_batch_many(std::span<const double>(xs + begin, cnt), k, tables,
                                    std::span<double>(out + begin * row, cnt * row));
          },
          nullptr, 0);
    });
    begin += cnt;
  }
  for (auto& t : pool) t.join();
  for (int s : status)
    if (s != kOk) return s;
  return kOk;
}

// boysfn::boys_batch_region (eval.hpp:39-41): region 0/1/2 = A/B/C.
int ref_boys_batch_region(double x, int k, int region, double* out, char* msg, size_t msg_len) {
  return guarded(
      [&] {
        const auto b = boysfn::boys_batch_region(x, k, boysfn::embedded_default(),
                                                 static_cast<boysfn::Region>(region));
        std::memcpy(out, b.values.data(), b.values.size() * sizeof(double));
      },
      msg, msg_len);
}

// boysfn::classify_region (eval.hpp:23).
int ref_classify_region(double x) {
  return static_cast<int>(boysfn::classify_region(x, boysfn::embedded_default()));
}

// emit_tables(embedded_default()) (tables.cpp:146-160).  Returns the length;
// writes at most len-1 characters plus a terminator.
size_t ref_emit_embedded(char* buf, size_t len) {
  const std::string s = boysfn::emit_tables(boysfn::embedded_default());
  if (buf && len) copy_msg(s.c_str(), buf, len);
  return s.size();
}

// emit_tables(parse_tables(text)) (tables.cpp:79-160), or the error message.
int ref_parse_emit(const char* text, char* buf, size_t len) {
  return guarded(
      [&] {
        const std::string s = boysfn::emit_tables(boysfn::parse_tables(text));
        copy_msg(s.c_str(), buf, len);
      },
      buf, len);
}

}  // extern "C"
