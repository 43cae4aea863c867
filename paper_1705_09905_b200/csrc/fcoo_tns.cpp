// fcoo_tns.cpp — FROSTT .tns text reader / writer (host only; declared in include/fcoo.h).
//
// Table IV's tensors (FROSTT) are distributed as text, one nonzero per line,
// "i_1 ... i_N v" with 1-based coordinates.  The reader maps the whole file into one buffer,
// cuts it into per-thread chunks at line boundaries, parses each chunk with std::from_chars
// (coordinates as integers, the value rounded once to fp32), and concatenates the chunks in
// file order.  Malformed input is reported with its 1-based line number, never skipped.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "fcoo_internal.cuh"

struct fcoo_tns_s {
  int order = 0;
  int64_t dims[fcoo::kMaxOrder] = {0};
  int64_t nnz = 0;
  std::vector<uint32_t> idx[fcoo::kMaxOrder];  // 0-based
  std::vector<float> val;
};

namespace {

using fcoo::kMaxOrder;

inline bool is_blank(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

enum LineKind { kSkip, kData, kBad };

// Parse the line [p, eol).  Returns kSkip for blank / comment lines, kData with the coordinates
// (1-based, checked to [1, 2^32-1]) and value on success, kBad otherwise.  With order == 0 it
// only counts the fields (into *fields) to fix the arity from the first data line.
LineKind parse_line(const char* p, const char* eol, int order, uint64_t* c, float* v, int* fields) {
  while (p < eol && is_blank(*p)) ++p;
  if (p == eol || *p == '#') return kSkip;
  if (order == 0) {
    int n = 0;
    while (p < eol) {
      ++n;
      while (p < eol && !is_blank(*p)) ++p;
      while (p < eol && is_blank(*p)) ++p;
    }
    *fields = n;
    return kData;
  }
  for (int m = 0; m < order; ++m) {
    uint64_t x = 0;
    auto r = std::from_chars(p, eol, x);
    if (r.ec != std::errc() || r.ptr == eol || !is_blank(*r.ptr) || x < 1 || x > 0xFFFFFFFFull) return kBad;
    c[m] = x;
    p = r.ptr;
    while (p < eol && is_blank(*p)) ++p;
  }
  if (p == eol) return kBad;  // value missing
  float f = 0.f;
  auto r = std::from_chars(p, eol, f);
  if (r.ec != std::errc()) return kBad;
  p = r.ptr;
  while (p < eol && is_blank(*p)) ++p;
  if (p != eol) return kBad;  // trailing field
  *v = f;
  return kData;
}

struct Chunk {
  std::vector<uint32_t> idx;  // order x count, interleaved per nonzero
  std::vector<float> val;
  uint64_t maxc[kMaxOrder] = {0};
  int64_t bad_at = -1;  // byte offset of the first malformed line
};

void parse_chunk(const char* buf, size_t b, size_t e, int order, Chunk* out) {
  uint64_t c[kMaxOrder];
  float v;
  size_t p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(memchr(buf + p, '\n', e - p));
    size_t eol = nl ? (size_t)(nl - buf) : e;
    LineKind k = parse_line(buf + p, buf + eol, order, c, &v, nullptr);
    if (k == kBad) { out->bad_at = (int64_t)p; return; }
    if (k == kData) {
      for (int m = 0; m < order; ++m) {
        out->idx.push_back((uint32_t)(c[m] - 1));
        out->maxc[m] = std::max(out->maxc[m], c[m]);
      }
      out->val.push_back(v);
    }
    p = eol + 1;
  }
}

int64_t line_number(const char* buf, size_t off) {
  return 1 + (int64_t)std::count(buf, buf + off, '\n');
}

}  // namespace

extern "C" {

fcoo_status fcoo_tns_read(const char* path, int nthreads, const int64_t* dims_override, fcoo_tns_t* out) {
  using fcoo::fail;
  if (!path || !out) return fail(FCOO_ERR_ARG, "NULL path/out");
  *out = nullptr;
  FILE* fp = fopen(path, "rb");
  if (!fp) return fail(FCOO_ERR_IO, "cannot open %s", path);
  std::vector<char> buf;
  if (fseek(fp, 0, SEEK_END) == 0) {
    long sz = ftell(fp);
    if (sz > 0) {
      buf.resize((size_t)sz);
      rewind(fp);
      if (fread(buf.data(), 1, buf.size(), fp) != buf.size()) { fclose(fp); return fail(FCOO_ERR_IO, "short read of %s", path); }
    }
  }
  fclose(fp);
  const size_t n = buf.size();
  const char* B = buf.data();

  // arity from the first data line
  int order = 0;
  for (size_t p = 0; p < n;) {
    const char* nl = static_cast<const char*>(memchr(B + p, '\n', n - p));
    size_t eol = nl ? (size_t)(nl - B) : n;
    int fields = 0;
    if (parse_line(B + p, B + eol, 0, nullptr, nullptr, &fields) == kData) { order = fields - 1; break; }
    p = eol + 1;
  }
  if (order == 0) return fail(FCOO_ERR_EMPTY, "%s: no data lines", path);
  if (order < 2 || order > kMaxOrder) return fail(FCOO_ERR_ORDER, "%s: %d coordinates per line, need 2..8", path, order);

  // per-thread chunks cut at line starts (>= 1 MB each)
  int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::max<size_t>(1, std::min<size_t>((size_t)nt, n / (1u << 20) + 1));
  std::vector<size_t> cut(nt + 1, n);
  cut[0] = 0;
  for (int k = 1; k < nt; ++k) {
    size_t p = std::max(cut[k - 1], n / nt * k);
    while (p < n && p > 0 && B[p - 1] != '\n') ++p;
    cut[k] = p;
  }
  std::vector<Chunk> ch(nt);
  {
    std::vector<std::thread> th;
    for (int k = 1; k < nt; ++k) th.emplace_back(parse_chunk, B, cut[k], cut[k + 1], order, &ch[k]);
    parse_chunk(B, cut[0], cut[1], order, &ch[0]);
    for (auto& t : th) t.join();
  }
  for (int k = 0; k < nt; ++k)
    if (ch[k].bad_at >= 0)
      return fail(FCOO_ERR_IO, "%s:%lld: malformed line (need %d positive integer coordinates < 2^32 and a value)",
                  path, (long long)line_number(B, (size_t)ch[k].bad_at), order);

  int64_t nnz = 0;
  uint64_t maxc[kMaxOrder] = {0};
  for (auto& c : ch) {
    nnz += (int64_t)c.val.size();
    for (int m = 0; m < order; ++m) maxc[m] = std::max(maxc[m], c.maxc[m]);
  }
  if (nnz == 0) return fail(FCOO_ERR_EMPTY, "%s: no data lines", path);
  fcoo_tns_s* t = new fcoo_tns_s;
  t->order = order;
  t->nnz = nnz;
  for (int m = 0; m < order; ++m) {
    if (dims_override) {
      if (dims_override[m] < 1 || dims_override[m] > 4294967295LL) {
        delete t;
        return fail(FCOO_ERR_ARG, "dims_override[%d]=%lld outside [1, 2^32)", m, (long long)dims_override[m]);
      }
      if ((int64_t)maxc[m] > dims_override[m]) {
        delete t;
        return fail(FCOO_ERR_INDEX_RANGE, "%s: mode %d coordinate %llu > dims_override %lld", path, m,
                    (unsigned long long)maxc[m], (long long)dims_override[m]);
      }
      t->dims[m] = dims_override[m];
    } else {
      t->dims[m] = (int64_t)maxc[m];
    }
    t->idx[m].resize((size_t)nnz);
  }
  t->val.resize((size_t)nnz);
  int64_t base = 0;
  for (auto& c : ch) {  // de-interleave in file order
    const int64_t cnt = (int64_t)c.val.size();
    for (int64_t q = 0; q < cnt; ++q)
      for (int m = 0; m < order; ++m) t->idx[m][(size_t)(base + q)] = c.idx[(size_t)(q * order + m)];
    std::copy(c.val.begin(), c.val.end(), t->val.begin() + base);
    base += cnt;
  }
  *out = t;
  return FCOO_OK;
}

fcoo_status fcoo_tns_info(fcoo_tns_t t, int* order, int64_t* dims, int64_t* nnz) {
  if (!t) return fcoo::fail(FCOO_ERR_ARG, "NULL tensor");
  if (order) *order = t->order;
  if (dims) for (int m = 0; m < t->order; ++m) dims[m] = t->dims[m];
  if (nnz) *nnz = t->nnz;
  return FCOO_OK;
}

fcoo_status fcoo_tns_copy(fcoo_tns_t t, uint32_t* const* idx, float* val) {
  if (!t || !idx || !val) return fcoo::fail(FCOO_ERR_ARG, "NULL tensor/idx/val");
  for (int m = 0; m < t->order; ++m) {
    if (!idx[m]) return fcoo::fail(FCOO_ERR_ARG, "idx[%d] is NULL", m);
    memcpy(idx[m], t->idx[m].data(), sizeof(uint32_t) * (size_t)t->nnz);
  }
  memcpy(val, t->val.data(), sizeof(float) * (size_t)t->nnz);
  return FCOO_OK;
}

fcoo_status fcoo_tns_destroy(fcoo_tns_t t) {
  delete t;
  return FCOO_OK;
}

fcoo_status fcoo_tns_write(const char* path, int order, int64_t nnz, const uint32_t* const* idx, const float* val) {
  using fcoo::fail;
  if (!path || (nnz > 0 && (!idx || !val))) return fail(FCOO_ERR_ARG, "NULL path/idx/val");
  if (order < 2 || order > kMaxOrder) return fail(FCOO_ERR_ORDER, "order %d outside [2,8]", order);
  if (nnz < 0) return fail(FCOO_ERR_ARG, "nnz < 0");
  for (int m = 0; m < order && nnz > 0; ++m) if (!idx[m]) return fail(FCOO_ERR_ARG, "idx[%d] is NULL", m);
  FILE* fp = fopen(path, "wb");
  if (!fp) return fail(FCOO_ERR_IO, "cannot create %s", path);
  std::vector<char> out;
  out.reserve(1 << 22);
  char tmp[64];
  bool ok = true;
  for (int64_t q = 0; q < nnz && ok; ++q) {
    for (int m = 0; m < order; ++m) {
      auto r = std::to_chars(tmp, tmp + sizeof(tmp), (uint64_t)idx[m][q] + 1);
      out.insert(out.end(), tmp, r.ptr);
      out.push_back(' ');
    }
    int k = snprintf(tmp, sizeof(tmp), "%.9g\n", (double)val[q]);
    out.insert(out.end(), tmp, tmp + k);
    if (out.size() >= (1u << 22)) {
      ok = fwrite(out.data(), 1, out.size(), fp) == out.size();
      out.clear();
    }
  }
  if (ok && !out.empty()) ok = fwrite(out.data(), 1, out.size(), fp) == out.size();
  if (fclose(fp) != 0) ok = false;
  return ok ? FCOO_OK : fail(FCOO_ERR_IO, "write to %s failed", path);
}

}  // extern "C"
