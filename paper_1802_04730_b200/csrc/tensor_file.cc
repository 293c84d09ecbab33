// tensor_file.cc — TCTN1 tensor files, byte-compatible with the reference's
// writeTensorFile / readTensorFile (proj/src/support/tensor_data.cc:122-189,
// format in proj/include/tc/support/tensor_data.h:52-60):
//   "TCTN1", kind byte 'f' | 'i', rank byte (<= 16),
//   rank x uint64 little-endian extents (each >= 1),
//   volume x 4-byte little-endian values (fp32 bits or int32).
// Failures are ErrorKind::Io with the reference's messages. tc-b200 tensors
// carry at most TCB_MAX_RANK (8) dimensions; a valid file of higher rank is
// rejected with Io as well.
#include "tensor_file.h"

#include <cstring>
#include <fstream>

namespace tcb {

namespace {

const char kMagic[5] = {'T', 'C', 'T', 'N', '1'};

void putU32(std::ostream& os, uint32_t v) {
  char b[4];
  for (int i = 0; i < 4; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
  os.write(b, 4);
}
void putU64(std::ostream& os, uint64_t v) {
  char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
  os.write(b, 8);
}
uint64_t getLE(std::istream& is, int n) {
  unsigned char b[8] = {0};
  is.read(reinterpret_cast<char*>(b), n);
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}

}  // namespace

void writeTensorFile(const std::string& path, const TensorFile& t) {
  std::ofstream os(path, std::ios::binary);
  if (!os) fail(ErrorKind::Io, "cannot open '" + path + "' for writing");
  os.write(kMagic, sizeof(kMagic));
  os.put(t.isInt ? 'i' : 'f');
  os.put(static_cast<char>(t.shape.size()));
  for (int64_t e : t.shape) putU64(os, static_cast<uint64_t>(e));
  for (uint32_t bits : t.bits) putU32(os, bits);
  if (!os) fail(ErrorKind::Io, "write failed for '" + path + "'");
}

TensorFile readTensorFile(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(ErrorKind::Io, "cannot open '" + path + "' for reading");
  char magic[5];
  is.read(magic, 5);
  if (!is || std::memcmp(magic, kMagic, 5) != 0) fail(ErrorKind::Io, "'" + path + "' is not a TCTN1 tensor file");
  int kind = is.get();
  int rank = is.get();
  if (!is || (kind != 'f' && kind != 'i') || rank < 0 || rank > 16)
    fail(ErrorKind::Io, "'" + path + "' has a malformed tensor header");
  TensorFile t;
  t.isInt = kind == 'i';
  int64_t n = 1;
  for (int d = 0; d < rank; ++d) {
    int64_t e = static_cast<int64_t>(getLE(is, 8));
    if (!is || e < 1) fail(ErrorKind::Io, "'" + path + "' declares an empty tensor extent");
    t.shape.push_back(e);
    n *= e;
  }
  if (rank > 8) fail(ErrorKind::Io, "'" + path + "' has rank " + std::to_string(rank) + " (tc-b200 tensors have at most 8)");
  t.bits.resize(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) {
    uint32_t v = static_cast<uint32_t>(getLE(is, 4));
    if (!is) fail(ErrorKind::Io, "'" + path + "' is truncated");
    t.bits[static_cast<size_t>(k)] = v;
  }
  return t;
}

}  // namespace tcb
