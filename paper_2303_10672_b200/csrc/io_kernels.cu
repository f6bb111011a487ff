// Policy CSV on the device (runner.cpp:90-166 policy_to_csv /
// policy_from_csv, io.cpp:53-92 parse_csv).  The >16M-state policy of
// b/m3/exp1 is a 320 MB CSV: formatting it row by row on the host costs tens
// of seconds, next to a 0.09 s solve.  Here one thread formats / parses one
// row: row lengths -> exclusive scan (CUB) -> byte offsets -> rows written in
// place; parsing finds the line ends with a CUB select, parses every row in
// parallel and reproduces the reference's error order (the first bad row in
// file order wins; field count, then numeric, then tuple range) and its
// last-row-wins rule for duplicate states.
#include <cub/cub.cuh>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "engine.hpp"

namespace pvi_b200 {
namespace {

__device__ __forceinline__ int n_digits_u32(std::uint32_t v) {
  int n = 1;
  while (v >= 10u) {
    v /= 10u;
    ++n;
  }
  return n;
}

__device__ __forceinline__ char* put_u32(char* p, std::uint32_t v, int nd) {
  for (int i = nd - 1; i >= 0; --i) {
    p[i] = static_cast<char>('0' + v % 10u);
    v /= 10u;
  }
  return p + nd;
}

// decode(s) then the action fields (append_action_fields): B writes the
// pair (a / (A_b + 1), a % (A_b + 1)), A and C the action itself.
template <bool WRITE>
__global__ void k_csv_rows(DevModel dm, const std::uint32_t* __restrict__ act, std::uint64_t n,
                           std::uint32_t nb, std::uint64_t* __restrict__ len,
                           const std::uint64_t* __restrict__ off, char* __restrict__ out) {
  const std::uint64_t s = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  std::uint64_t rem = s;
  std::uint32_t fields[kMaxDigits + 2];
  int nf = 0;
  for (int i = 0; i < dm.n_digits; ++i) {
    fields[nf++] = static_cast<std::uint32_t>(rem / dm.weight[i]);
    rem %= dm.weight[i];
  }
  const std::uint32_t a = act[s];
  if (nb) {
    fields[nf++] = a / nb;
    fields[nf++] = a % nb;
  } else {
    fields[nf++] = a;
  }
  if (!WRITE) {
    std::uint64_t l = 0;
    for (int i = 0; i < nf; ++i) l += n_digits_u32(fields[i]) + 1;  // digits + ',' or '\n'
    len[s] = l;
    return;
  }
  char* p = out + off[s];
  for (int i = 0; i < nf; ++i) {
    p = put_u32(p, fields[i], n_digits_u32(fields[i]));
    *p++ = i + 1 < nf ? ',' : '\n';
  }
}

struct IsNewline {
  const char* t;
  __device__ bool operator()(std::uint64_t i) const { return t[i] == '\n'; }
};

// std::stoi on one field with the '\r' of the row removed (parse_csv drops
// them): leading whitespace, optional sign, >= 1 digit, stop at the first
// other character; false when nothing converts or the value leaves int.
__device__ bool field_stoi(const char* t, std::uint64_t a, std::uint64_t b, int* out) {
  std::uint64_t i = a;
  auto skip_cr = [&] {
    while (i < b && t[i] == '\r') ++i;
  };
  skip_cr();
  while (i < b && (t[i] == ' ' || t[i] == '\t' || t[i] == '\v' || t[i] == '\f')) {
    ++i;
    skip_cr();
  }
  bool neg = false;
  if (i < b && (t[i] == '+' || t[i] == '-')) {
    neg = t[i] == '-';
    ++i;
    skip_cr();
  }
  long long v = 0;
  int nd = 0;
  while (i < b && t[i] >= '0' && t[i] <= '9') {
    v = v * 10 + (t[i] - '0');
    if (v > 2147483648ll) return false;
    ++nd;
    ++i;
    skip_cr();
  }
  if (nd == 0) return false;
  if (neg) v = -v;
  if (v > 2147483647ll || v < -2147483648ll) return false;
  *out = static_cast<int>(v);
  return true;
}

// Row r (1-based, the header is row 0) spans [start(r), end(r)).
// err: min over bad rows of (r << 2 | code), code 1 field count, 2 numeric,
// 3 tuple range.  owner[state] = last row naming the state.
__global__ void k_csv_parse(DevModel dm, const char* __restrict__ t, const std::uint64_t* __restrict__ nl,
                            std::uint64_t n_rows_body, std::uint64_t text_len, int n_cols, std::uint32_t nb,
                            unsigned long long* __restrict__ err, unsigned long long* __restrict__ owner,
                            std::uint64_t* __restrict__ row_state, std::uint32_t* __restrict__ row_act) {
  const std::uint64_t k = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n_rows_body) return;
  const std::uint64_t r = k + 1;
  const std::uint64_t a = nl[r - 1] + 1;
  const std::uint64_t b = r < n_rows_body + 1 && nl[r] != ~0ull ? nl[r] : text_len;
  // field count
  int nf = 1;
  for (std::uint64_t i = a; i < b; ++i) nf += t[i] == ',';
  const unsigned long long key = static_cast<unsigned long long>(r) << 2;
  if (nf != n_cols) {
    atomicMin(err, key | 1ull);
    return;
  }
  int vals[kMaxDigits + 2];
  std::uint64_t fa = a;
  int f = 0;
  for (std::uint64_t i = a; i <= b; ++i) {
    if (i == b || t[i] == ',') {
      if (!field_stoi(t, fa, i, &vals[f])) {
        atomicMin(err, key | 2ull);
        return;
      }
      ++f;
      fa = i + 1;
    }
  }
  std::uint64_t idx = 0;
  for (int i = 0; i < dm.n_digits; ++i) {
    if (vals[i] < 0 || vals[i] >= dm.radix[i]) {
      atomicMin(err, key | 3ull);
      return;
    }
    idx += static_cast<std::uint64_t>(vals[i]) * dm.weight[i];
  }
  const int d = dm.n_digits;
  const std::uint32_t act = nb ? static_cast<std::uint32_t>(vals[d] * static_cast<int>(nb) + vals[d + 1])
                               : static_cast<std::uint32_t>(vals[d]);
  row_state[k] = idx;
  row_act[k] = act;
  atomicMax(owner + idx, static_cast<unsigned long long>(r));
}

__global__ void k_csv_scatter(std::uint64_t n_rows_body, const std::uint64_t* __restrict__ row_state,
                              const std::uint32_t* __restrict__ row_act,
                              const unsigned long long* __restrict__ owner, std::uint32_t* __restrict__ out) {
  const std::uint64_t k = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n_rows_body) return;
  const std::uint64_t s = row_state[k];
  if (owner[s] == k + 1) out[s] = row_act[k];
}

unsigned grid1(std::uint64_t n, unsigned block) { return static_cast<unsigned>((n + block - 1) / block); }

struct CsvStream {
  cudaStream_t s = nullptr;
  CsvStream() { PVI_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~CsvStream() {
    if (s) cudaStreamDestroy(s);
  }
};

}  // namespace

std::uint64_t policy_csv_format(const Model& m, const std::uint32_t* actions, char* out,
                                std::uint64_t capacity) {
  if (m.scenario == PVI_TABULAR) fail(PVI_ERR_PARAMETER, "tabular models have no policy CSV");
  const int device = select_device(-1);
  const DevModel& dm = m.device_view(device);
  const std::uint64_t n = m.space.count;
  const std::uint32_t nb = m.scenario == PVI_SCENARIO_B ? static_cast<std::uint32_t>(m.b_nb) : 0u;
  CsvStream cs;
  cudaStream_t st = cs.s;
  PoolBuf dact(n * 4, st), dlen((n + 1) * 8, st), doff((n + 1) * 8, st);
  PVI_CUDA(cudaMemcpyAsync(dact.p, actions, n * 4, cudaMemcpyHostToDevice, st));
  // row lengths, then one exclusive scan over n + 1 entries: off[n] = total
  PVI_CUDA(cudaMemsetAsync(dlen.as<std::uint64_t>() + n, 0, 8, st));
  k_csv_rows<false><<<grid1(n, 256), 256, 0, st>>>(dm, dact.as<std::uint32_t>(), n, nb, dlen.as<std::uint64_t>(),
                                                    nullptr, nullptr);
  PVI_CUDA(cudaGetLastError());
  std::size_t tmp_bytes = 0;
  PVI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, dlen.as<std::uint64_t>(), doff.as<std::uint64_t>(),
                                         n + 1, st));
  PoolBuf tmp(tmp_bytes, st);
  PVI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, dlen.as<std::uint64_t>(), doff.as<std::uint64_t>(),
                                         n + 1, st));
  std::uint64_t total = 0;
  PVI_CUDA(cudaMemcpyAsync(&total, doff.as<std::uint64_t>() + n, 8, cudaMemcpyDeviceToHost, st));
  PVI_CUDA(cudaStreamSynchronize(st));
  if (!out) return total;
  if (capacity < total) fail(PVI_ERR_PARAMETER, "policy CSV buffer too small");
  PoolBuf dout(total, st);
  k_csv_rows<true><<<grid1(n, 256), 256, 0, st>>>(dm, dact.as<std::uint32_t>(), n, nb, nullptr,
                                                   doff.as<std::uint64_t>(), dout.as<char>());
  PVI_CUDA(cudaGetLastError());
  PVI_CUDA(cudaMemcpyAsync(out, dout.p, total, cudaMemcpyDeviceToHost, st));
  PVI_CUDA(cudaStreamSynchronize(st));
  return total;
}

// policy_from_csv after the metadata check: the whole file text in, the
// policy out, or the reference's FormatError / IndexingError.  Quoted CSV
// (never written by either runner) goes through the host restatement of
// parse_csv instead, with the same checks.
namespace {

void parse_host_quoted(const Model& m, const char* text, std::uint64_t len, std::uint32_t* out);

std::string row_text(const char* t, std::uint64_t a, std::uint64_t b) {
  std::string s;
  for (std::uint64_t i = a; i < b; ++i)
    if (t[i] != '\r') s += t[i];
  return s;
}

}  // namespace

void policy_csv_parse(const Model& m, const char* text, std::uint64_t len, std::uint32_t* out) {
  if (m.scenario == PVI_TABULAR) fail(PVI_ERR_PARAMETER, "tabular models have no policy CSV");
  const std::uint64_t n = m.space.count;
  const int arity = static_cast<int>(m.space.radix.size());
  const int n_cols = arity + (m.scenario == PVI_SCENARIO_B ? 2 : 1);
  const std::uint32_t nb = m.scenario == PVI_SCENARIO_B ? static_cast<std::uint32_t>(m.b_nb) : 0u;
  if (std::memchr(text, '"', len)) {
    parse_host_quoted(m, text, len, out);
    return;
  }
  const int device = select_device(-1);
  const DevModel& dm = m.device_view(device);
  CsvStream cs;
  cudaStream_t st = cs.s;
  PoolBuf dt(len + 1, st);
  PVI_CUDA(cudaMemcpyAsync(dt.p, text, len, cudaMemcpyHostToDevice, st));
  // line ends
  PoolBuf dnl((len + 1) * 8, st), dcount(8, st);
  std::size_t tmp_bytes = 0;
  cub::CountingInputIterator<std::uint64_t> it(0);
  IsNewline pred{dt.as<char>()};
  cub::DeviceSelect::If(nullptr, tmp_bytes, it, dnl.as<std::uint64_t>(), dcount.as<std::uint64_t>(), len, pred, st);
  PoolBuf tmp(tmp_bytes, st);
  PVI_CUDA(cub::DeviceSelect::If(tmp.p, tmp_bytes, it, dnl.as<std::uint64_t>(), dcount.as<std::uint64_t>(), len,
                                 pred, st));
  std::uint64_t n_nl = 0;
  PVI_CUDA(cudaMemcpyAsync(&n_nl, dcount.p, 8, cudaMemcpyDeviceToHost, st));
  PVI_CUDA(cudaStreamSynchronize(st));
  // rows as parse_csv counts them: one per '\n', plus a last row when text
  // other than '\r' follows the last '\n'
  std::vector<std::uint64_t> last_nl(1, 0);
  std::uint64_t tail_start = 0;
  if (n_nl) {
    PVI_CUDA(cudaMemcpy(&last_nl[0], dnl.as<std::uint64_t>() + n_nl - 1, 8, cudaMemcpyDeviceToHost));
    tail_start = last_nl[0] + 1;
  }
  bool tail_row = false;
  for (std::uint64_t i = tail_start; i < len; ++i)
    if (text[i] != '\r') {
      tail_row = true;
      break;
    }
  const std::uint64_t rows = n_nl + (tail_row ? 1 : 0);
  if (rows != n + 1)
    fail(PVI_ERR_FORMAT, "policy CSV has " + std::to_string(rows) + " rows, expected " + std::to_string(n + 1));
  // nl[n_nl] = ~0 marks "to the end of the text" for the tail row
  const std::uint64_t marker = ~0ull;
  PVI_CUDA(cudaMemcpyAsync(dnl.as<std::uint64_t>() + n_nl, &marker, 8, cudaMemcpyHostToDevice, st));
  PoolBuf derr(8, st), downer(n * 8, st), drs(n * 8, st), dra(n * 4, st), dout(n * 4, st);
  const unsigned long long none = ~0ull;
  PVI_CUDA(cudaMemcpyAsync(derr.p, &none, 8, cudaMemcpyHostToDevice, st));
  PVI_CUDA(cudaMemsetAsync(downer.p, 0, n * 8, st));
  PVI_CUDA(cudaMemsetAsync(dout.p, 0, n * 4, st));
  k_csv_parse<<<grid1(n, 256), 256, 0, st>>>(dm, dt.as<char>(), dnl.as<std::uint64_t>(), n, len, n_cols, nb,
                                              derr.as<unsigned long long>(), downer.as<unsigned long long>(),
                                              drs.as<std::uint64_t>(), dra.as<std::uint32_t>());
  PVI_CUDA(cudaGetLastError());
  unsigned long long e = 0;
  PVI_CUDA(cudaMemcpyAsync(&e, derr.p, 8, cudaMemcpyDeviceToHost, st));
  PVI_CUDA(cudaStreamSynchronize(st));
  if (e != ~0ull) {
    // the first bad row in file order: rebuild the reference's message
    const std::uint64_t r = e >> 2;
    std::uint64_t ab[2];
    PVI_CUDA(cudaMemcpy(ab, dnl.as<std::uint64_t>() + r - 1, 16, cudaMemcpyDeviceToHost));
    const std::uint64_t a = ab[0] + 1, b = ab[1] == ~0ull ? len : ab[1];
    const std::string row = row_text(text, a, b);
    std::vector<std::string> fields(1);
    for (char c : row) {
      if (c == ',') fields.emplace_back();
      else fields.back() += c;
    }
    switch (e & 3ull) {
      case 1:
        fail(PVI_ERR_FORMAT, "policy CSV row " + std::to_string(r) + " has " + std::to_string(fields.size()) +
                                 " fields");
      case 2:
        fail(PVI_ERR_FORMAT, "policy CSV row " + std::to_string(r) + " is not numeric");
      default:
        for (int i = 0; i < arity; ++i) {
          const int v = std::stoi(fields[i]);
          if (v < 0 || v >= m.space.radix[i])
            fail(PVI_ERR_INDEXING, "tuple component " + std::to_string(i) + " = " + std::to_string(v) +
                                       " outside [0, " + std::to_string(m.space.radix[i] - 1) + "]");
        }
        fail(PVI_ERR_INDEXING, "policy CSV row " + std::to_string(r) + " out of range");
    }
  }
  k_csv_scatter<<<grid1(n, 256), 256, 0, st>>>(n, drs.as<std::uint64_t>(), dra.as<std::uint32_t>(),
                                                downer.as<unsigned long long>(), dout.as<std::uint32_t>());
  PVI_CUDA(cudaGetLastError());
  PVI_CUDA(cudaMemcpyAsync(out, dout.p, n * 4, cudaMemcpyDeviceToHost, st));
  PVI_CUDA(cudaStreamSynchronize(st));
}

namespace {

// io.cpp:53-92 parse_csv + runner.cpp:110-148, for quoted input
void parse_host_quoted(const Model& m, const char* text, std::uint64_t len, std::uint32_t* out) {
  std::vector<std::vector<std::string>> rows;
  std::vector<std::string> row;
  std::string field;
  bool quoted = false;
  auto end_field = [&] {
    row.push_back(field);
    field.clear();
  };
  auto end_row = [&] {
    end_field();
    rows.push_back(row);
    row.clear();
  };
  for (std::uint64_t i = 0; i < len; ++i) {
    const char c = text[i];
    if (quoted) {
      if (c == '"') {
        if (i + 1 < len && text[i + 1] == '"') {
          field += '"';
          ++i;
        } else {
          quoted = false;
        }
      } else {
        field += c;
      }
    } else if (c == '"') {
      quoted = true;
    } else if (c == ',') {
      end_field();
    } else if (c == '\n') {
      end_row();
    } else if (c != '\r') {
      field += c;
    }
  }
  if (!field.empty() || !row.empty()) end_row();
  const std::uint64_t n = m.space.count;
  const std::size_t arity = m.space.radix.size();
  const std::size_t n_cols = arity + (m.scenario == PVI_SCENARIO_B ? 2 : 1);
  if (rows.size() != n + 1)
    fail(PVI_ERR_FORMAT, "policy CSV has " + std::to_string(rows.size()) + " rows, expected " +
                             std::to_string(n + 1));
  std::memset(out, 0, n * 4);
  std::vector<int> v(n_cols);
  for (std::size_t r = 1; r < rows.size(); ++r) {
    if (rows[r].size() != n_cols)
      fail(PVI_ERR_FORMAT, "policy CSV row " + std::to_string(r) + " has " + std::to_string(rows[r].size()) +
                               " fields");
    try {
      for (std::size_t i = 0; i < n_cols; ++i) v[i] = std::stoi(rows[r][i]);
    } catch (const std::exception&) {
      fail(PVI_ERR_FORMAT, "policy CSV row " + std::to_string(r) + " is not numeric");
    }
    std::uint64_t idx = 0;
    for (std::size_t i = 0; i < arity; ++i) {
      if (v[i] < 0 || v[i] >= m.space.radix[i])
        fail(PVI_ERR_INDEXING, "tuple component " + std::to_string(i) + " = " + std::to_string(v[i]) +
                                   " outside [0, " + std::to_string(m.space.radix[i] - 1) + "]");
      idx += static_cast<std::uint64_t>(v[i]) * m.space.weight[i];
    }
    out[idx] = m.scenario == PVI_SCENARIO_B ? static_cast<std::uint32_t>(v[arity] * m.b_nb + v[arity + 1])
                                            : static_cast<std::uint32_t>(v[arity]);
  }
}

}  // namespace
}  // namespace pvi_b200
