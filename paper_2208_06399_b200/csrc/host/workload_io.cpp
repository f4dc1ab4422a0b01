// Pool and workload files in the reference format (workload_io.hpp:14-26):
// a line-oriented text header, then per table (ascending id)
//   u64 n_offsets, i64 offsets[n_offsets], u64 n_indices, i64 indices[n_indices]
// little-endian. Validation and error classes follow load_workload
// (workload_io.hpp:178-245): OffsetError / IndexError naming "table <id>".
// Arrays are moved in bulk (the host is little-endian x86-64), not per value.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "host.hpp"

namespace asb {
namespace {

std::string fmt_double(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::string header_line(const as_table_spec& t) {
  std::ostringstream os;
  os << "table " << t.id << ' ' << t.dim << ' ' << t.hash_size << ' ' << fmt_double(t.pooling_mean)
     << ' ' << fmt_double(t.access_ratio) << ' ' << t.bytes_per_param;
  return os.str();
}

as_table_spec parse_header_line(const std::string& line) {
  std::istringstream is(line);
  std::string tag;
  as_table_spec t;
  std::memset(&t, 0, sizeof t);
  long long hash = 0;
  if (!(is >> tag >> t.id >> t.dim >> hash >> t.pooling_mean >> t.access_ratio >> t.bytes_per_param) ||
      tag != "table")
    fail(AS_PARSE, "malformed table header line: '" + line + "'");
  t.hash_size = hash;
  if (t.dim < 1 || t.hash_size < 1 || t.bytes_per_param < 1)
    fail(AS_PARSE, "table " + std::to_string(t.id) + ": non-positive dim/hash_size/bytes_per_param");
  return t;
}

std::string get_line(std::istream& is, const std::string& what) {
  std::string line;
  if (!std::getline(is, line)) fail(AS_PARSE, "truncated file while reading " + what);
  if (!line.empty() && line.back() == '\r') line.pop_back();
  return line;
}

uint64_t get_u64(std::istream& is, const std::string& what) {
  unsigned char b[8];
  if (!is.read(reinterpret_cast<char*>(b), 8)) fail(AS_PARSE, "truncated file while reading " + what);
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
  return v;
}

void get_i64s(std::istream& is, int64_t* dst, uint64_t n, const std::string& what) {
  const std::streamsize bytes = static_cast<std::streamsize>(n * 8);
  if (bytes && !is.read(reinterpret_cast<char*>(dst), bytes))
    fail(AS_PARSE, "truncated file while reading " + what);
}

void put_u64(std::ostream& os, uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
  os.write(reinterpret_cast<const char*>(b), 8);
}

std::vector<as_table_spec> read_tables(std::istream& is, size_t count) {
  std::vector<as_table_spec> out;
  int last = -1;
  for (size_t i = 0; i < count; ++i) {
    as_table_spec t = parse_header_line(get_line(is, "table header"));
    if (t.id <= last) fail(AS_PARSE, "table " + std::to_string(t.id) + ": ids must be strictly ascending");
    last = t.id;
    out.push_back(t);
  }
  if (get_line(is, "end_header") != "end_header") fail(AS_PARSE, "missing end_header");
  return out;
}

}  // namespace

void save_pool(const std::string& path, const std::vector<as_table_spec>& tables) {
  std::ofstream os(path, std::ios::binary);
  if (!os) fail(AS_PARSE, "cannot open for writing: " + path);
  os << "autoshard-pool 1\ntables " << tables.size() << "\n";
  for (const auto& t : tables) os << header_line(t) << "\n";
  os << "end_header\n";
  if (!os) fail(AS_PARSE, "failed writing pool stream");
}

std::vector<as_table_spec> load_pool(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(AS_PARSE, "cannot open: " + path);
  const std::string magic = get_line(is, "pool magic");
  if (magic != "autoshard-pool 1") fail(AS_PARSE, "bad pool magic/version: '" + magic + "'");
  std::istringstream tl(get_line(is, "pool table count"));
  std::string tag;
  size_t count = 0;
  if (!(tl >> tag >> count) || tag != "tables") fail(AS_PARSE, "malformed pool table count line");
  return read_tables(is, count);
}

void save_workload(const std::string& path, const HostWorkload& wl,
                   const std::vector<as_table_spec>& tables) {
  if (tables.size() != wl.per_table.size())
    fail(AS_CONFIG, "save_workload: table metadata must match streams");
  std::ofstream os(path, std::ios::binary);
  if (!os) fail(AS_PARSE, "cannot open for writing: " + path);
  os << "autoshard-workload 1\nbatch_size " << wl.batch_size << "\ntables " << wl.per_table.size() << "\n";
  for (size_t i = 0; i < tables.size(); ++i) {
    if (tables[i].id != wl.per_table[i].table_id)
      fail(AS_CONFIG, "save_workload: metadata order must match streams");
    os << header_line(tables[i]) << "\n";
  }
  os << "end_header\n";
  for (const auto& s : wl.per_table) {
    put_u64(os, s.offsets.size());
    os.write(reinterpret_cast<const char*>(s.offsets.data()),
             static_cast<std::streamsize>(s.offsets.size() * 8));
    put_u64(os, s.indices.size());
    os.write(reinterpret_cast<const char*>(s.indices.data()),
             static_cast<std::streamsize>(s.indices.size() * 8));
  }
  if (!os) fail(AS_PARSE, "failed writing workload stream");
}

void load_workload(const std::string& path, HostWorkload* wl, std::vector<as_table_spec>* tables) {
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(AS_PARSE, "cannot open: " + path);
  const std::string magic = get_line(is, "workload magic");
  if (magic != "autoshard-workload 1") fail(AS_PARSE, "bad workload magic/version: '" + magic + "'");
  std::string tag;
  {
    std::istringstream bl(get_line(is, "batch_size"));
    if (!(bl >> tag >> wl->batch_size) || tag != "batch_size" || wl->batch_size < 1)
      fail(AS_PARSE, "malformed batch_size line");
  }
  size_t count = 0;
  {
    std::istringstream tl(get_line(is, "table count"));
    if (!(tl >> tag >> count) || tag != "tables") fail(AS_PARSE, "malformed tables count line");
  }
  *tables = read_tables(is, count);
  wl->per_table.assign(count, HostStream{});
  for (size_t i = 0; i < count; ++i) {
    const as_table_spec& t = (*tables)[i];
    const std::string where = "table " + std::to_string(t.id);
    HostStream& s = wl->per_table[i];
    s.table_id = t.id;
    const uint64_t n_off = get_u64(is, where + " offset count");
    if (n_off != static_cast<uint64_t>(wl->batch_size) + 1)
      fail(AS_OFFSET, where + ": offsets length " + std::to_string(n_off) + " != batch_size + 1");
    s.offsets.resize(n_off);
    get_i64s(is, s.offsets.data(), n_off, where + " offsets");
    if (s.offsets.front() != 0)
      fail(AS_OFFSET, where + ": offsets must start at 0, got " + std::to_string(s.offsets.front()));
    for (size_t q = 1; q < s.offsets.size(); ++q)
      if (s.offsets[q] < s.offsets[q - 1])
        fail(AS_OFFSET, where + ": offsets must be nondecreasing at entry " + std::to_string(q));
    const uint64_t n_idx = get_u64(is, where + " index count");
    if (static_cast<int64_t>(n_idx) != s.offsets.back())
      fail(AS_OFFSET, where + ": final offset " + std::to_string(s.offsets.back()) +
                          " != index count " + std::to_string(n_idx));
    s.indices.resize(n_idx);
    // The reference validates index by index while reading, so an
    // out-of-range value before a truncation point wins over the truncation.
    is.read(reinterpret_cast<char*>(s.indices.data()), static_cast<std::streamsize>(n_idx * 8));
    const uint64_t got = static_cast<uint64_t>(is.gcount()) / 8;
    for (uint64_t q = 0; q < got; ++q) {
      const int64_t v = s.indices[q];
      if (v < 0 || v >= t.hash_size)
        fail(AS_INDEX, where + ": index " + std::to_string(v) + " out of range [0, " +
                           std::to_string(t.hash_size) + ")");
    }
    if (got != n_idx) fail(AS_PARSE, "truncated file while reading " + where + " indices");
  }
}

}  // namespace asb
