// dfftb C++ shim, part 2: the reference's DTNS tensor files
// (/root/reference/proj/include/dfft/tensor_file.hpp, src/tensor_file.cpp)
// over the dfft.hpp carrier.  Same container, same error codes
// (BadMagic, TruncatedFile, DimMismatch), same semantics:
//   read_tensor  — every rank gets its block of the file in `dist`'s layout;
//                  a real file feeding a complex layout is promoted
//   write_tensor — the blocks of all ranks assembled into one row-major file
//                  (written by rank 0)
// Differences: read_tensor reads the file on every rank (one node, shared
// file system) instead of scattering from rank 0; write_tensor gathers with
// the shim Comm's all_gather.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "dfftb/dfft.hpp"

namespace dfftb::dfft {

enum class TensorElement : std::uint8_t { Real64 = 0, Complex64 = 1, Real32 = 2, Complex32 = 3 };

/// magic "DTNS", u32 version = 1, u8 element kind, u32 axis count, u64 dims,
/// little-endian row-major payload (tensor_file.hpp:21-41)
struct TensorFile {
  GlobalDims dims;
  TensorElement element = TensorElement::Real64;
  std::vector<std::byte> payload;

  std::size_t element_bytes() const {
    switch (element) {
      case TensorElement::Real64: return 8;
      case TensorElement::Complex64: return 16;
      case TensorElement::Real32: return 4;
      case TensorElement::Complex32: return 8;
    }
    return 0;
  }
  bool is_complex() const { return element == TensorElement::Complex64 || element == TensorElement::Complex32; }
};

namespace detail {
inline Error tensor_error(ErrorCode c, const std::string& name, const std::string& what) {
  return Error(c, name + ": " + what);
}
}  // namespace detail

inline TensorFile read_tensor_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw detail::tensor_error(ErrorCode::TruncatedFile, "TruncatedFile", "cannot open " + path);
  char head[13];
  if (!f.read(head, 13)) throw detail::tensor_error(ErrorCode::TruncatedFile, "TruncatedFile", "unexpected end of " + path);
  if (std::memcmp(head, "DTNS", 4) != 0)
    throw detail::tensor_error(ErrorCode::BadMagic, "BadMagic", path + " is not a DTNS tensor");
  std::uint32_t version, axes;
  std::uint8_t kind;
  std::memcpy(&version, head + 4, 4);
  std::memcpy(&kind, head + 8, 1);
  std::memcpy(&axes, head + 9, 4);
  if (version != 1) throw detail::tensor_error(ErrorCode::BadMagic, "BadMagic", "unsupported DTNS version");
  if (kind > 3) throw detail::tensor_error(ErrorCode::BadMagic, "BadMagic", "unknown element kind");
  if (axes == 0 || axes > 16) throw detail::tensor_error(ErrorCode::BadMagic, "BadMagic", "implausible axis count");
  std::vector<std::int64_t> dims(axes);
  for (auto& d : dims) {
    std::uint64_t v;
    if (!f.read(reinterpret_cast<char*>(&v), 8))
      throw detail::tensor_error(ErrorCode::TruncatedFile, "TruncatedFile", "unexpected end of " + path);
    if (v < 1) throw detail::tensor_error(ErrorCode::BadMagic, "BadMagic", "non-positive axis length");
    d = static_cast<std::int64_t>(v);
  }
  TensorFile t;
  t.dims = GlobalDims(dims);
  t.element = static_cast<TensorElement>(kind);
  t.payload.resize(static_cast<std::size_t>(t.dims.total()) * t.element_bytes());
  if (!f.read(reinterpret_cast<char*>(t.payload.data()), static_cast<std::streamsize>(t.payload.size())))
    throw detail::tensor_error(ErrorCode::TruncatedFile, "TruncatedFile", "unexpected end of " + path);
  return t;
}

inline void write_tensor_file(const std::string& path, const TensorFile& t) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw detail::tensor_error(ErrorCode::TruncatedFile, "TruncatedFile", "cannot create " + path);
  const std::uint32_t version = 1, axes = static_cast<std::uint32_t>(t.dims.ndim());
  const std::uint8_t kind = static_cast<std::uint8_t>(t.element);
  f.write("DTNS", 4);
  f.write(reinterpret_cast<const char*>(&version), 4);
  f.write(reinterpret_cast<const char*>(&kind), 1);
  f.write(reinterpret_cast<const char*>(&axes), 4);
  for (std::size_t a = 0; a < t.dims.ndim(); ++a) {
    const std::uint64_t d = static_cast<std::uint64_t>(t.dims[a]);
    f.write(reinterpret_cast<const char*>(&d), 8);
  }
  f.write(reinterpret_cast<const char*>(t.payload.data()), static_cast<std::streamsize>(t.payload.size()));
  if (!f) throw detail::tensor_error(ErrorCode::TruncatedFile, "TruncatedFile", "write failed: " + path);
}

namespace detail {
// visit this rank's block of `dist` in local row-major order with global flat indices
template <class F>
void for_each_local(const Distribution& dist, int rank, F&& fn) {
  const LocalExtents ext = dist.extents_of(rank);
  const std::size_t nd = dist.dims.ndim();
  std::vector<std::int64_t> idx(nd, 0);
  const std::int64_t count = ext.count();
  for (std::int64_t l = 0; l < count; ++l) {
    std::int64_t g = 0;
    for (std::size_t a = 0; a < nd; ++a) g = g * dist.dims[a] + ext.axes[a].offset + idx[a];
    fn(l, g);
    for (std::size_t a = nd; a-- > 0;) {
      if (++idx[a] < ext.axes[a].length) break;
      idx[a] = 0;
    }
  }
}

template <class S>
S load_le(const std::byte* p) {
  S v;
  std::memcpy(&v, p, sizeof(S));
  return v;
}
}  // namespace detail

/// read_tensor (tensor_file.hpp:48-112): this rank's block of the file
template <class T>
DistTensor<T> read_tensor(Comm& comm, const Distribution& dist, const std::string& path) {
  const TensorFile file = read_tensor_file(path);
  if (!(file.dims == dist.dims))
    throw detail::tensor_error(ErrorCode::DimMismatch, "DimMismatch", "tensor file dims do not match the layout");
  const bool real_layout = dist.element == ElementKind::Real;
  if (real_layout && file.is_complex())
    throw detail::tensor_error(ErrorCode::DimMismatch, "DimMismatch", "complex tensor file cannot feed a real layout");
  auto t = DistTensor<T>::zeros(dist, comm.rank());
  const std::byte* pl = file.payload.data();
  const std::size_t eb = file.element_bytes();
  detail::for_each_local(dist, comm.rank(), [&](std::int64_t l, std::int64_t g) {
    const std::byte* e = pl + static_cast<std::size_t>(g) * eb;
    double re = 0, im = 0;
    switch (file.element) {
      case TensorElement::Real64: re = detail::load_le<double>(e); break;
      case TensorElement::Real32: re = detail::load_le<float>(e); break;
      case TensorElement::Complex64: re = detail::load_le<double>(e); im = detail::load_le<double>(e + 8); break;
      case TensorElement::Complex32: re = detail::load_le<float>(e); im = detail::load_le<float>(e + 4); break;
    }
    if (real_layout) t.real[static_cast<std::size_t>(l)] = static_cast<T>(re);
    else t.cplx[static_cast<std::size_t>(l)] = cx<T>(static_cast<T>(re), static_cast<T>(im));
  });
  t.from_host();
  return t;
}

/// write_tensor (tensor_file.hpp:115-160): all ranks' blocks -> one file
/// (collective; rank 0 writes)
template <class T>
void write_tensor(Comm& comm, const DistTensor<T>& tensor, const std::string& path) {
  DistTensor<T> local = tensor;
  local.to_host();
  const bool real = tensor.dist.element == ElementKind::Real;
  const std::size_t esz = real ? sizeof(T) : sizeof(cx<T>);
  // fixed-size all-gather: pad every block to the largest one
  std::int64_t maxn = 0;
  for (int r = 0; r < comm.size(); ++r) maxn = std::max(maxn, tensor.dist.local_count(r));
  std::vector<unsigned char> mine(static_cast<std::size_t>(maxn) * esz, 0);
  const void* src = real ? static_cast<const void*>(local.real.data()) : static_cast<const void*>(local.cplx.data());
  if (!mine.empty() && local.local_size()) std::memcpy(mine.data(), src, local.local_size() * esz);
  const std::vector<unsigned char> all = comm.size() > 1 ? comm.all_gather(mine) : mine;
  if (comm.rank() != 0) return;
  TensorFile f;
  f.dims = tensor.dist.dims;
  f.element = real ? (sizeof(T) == 8 ? TensorElement::Real64 : TensorElement::Real32)
                   : (sizeof(T) == 8 ? TensorElement::Complex64 : TensorElement::Complex32);
  f.payload.resize(static_cast<std::size_t>(f.dims.total()) * esz);
  for (int r = 0; r < comm.size(); ++r) {
    const unsigned char* blk = all.data() + static_cast<std::size_t>(r) * mine.size();
    detail::for_each_local(tensor.dist, r, [&](std::int64_t l, std::int64_t g) {
      std::memcpy(f.payload.data() + static_cast<std::size_t>(g) * esz, blk + static_cast<std::size_t>(l) * esz, esz);
    });
  }
  write_tensor_file(path, f);
}

}  // namespace dfftb::dfft
