// rk_records.cu -- RNKY block records (reference: proj/src/block_record.cpp:51-144,
// proj/include/ranky/block_record.hpp): the per-block U*Sigma payload file that
// workers hand to the coordinator, byte-identical to the reference's writer:
//   "RNKY" | version u16 = 1 | block index u32 | rows u32 | k u32 |
//   rows*k IEEE-754 doubles (row-major) | CRC32 of the payload bytes (u32),
// all little-endian. Reader errors carry the reference's RecordError messages.
//
// The CRC32 (reflected 0xEDB88320, init and xorout 0xFFFFFFFF, as
// block_record.cpp:53-68) of device-resident payloads runs on the GPU: one CTA
// per record, each thread the CRC of its slice (table in shared memory), and
// the slices combined in a tree with crc(A||B) = x^(8|B|) * crc(A) + crc(B) over
// GF(2) mod P (the zlib crc32_combine identity; the init/xorout terms cancel).
// Byte work, HBM-bound: every payload byte is read once.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "rk_internal.cuh"

namespace rk {
namespace {

constexpr uint32_t kPoly = 0xEDB88320u;

uint32_t host_table[256];
bool host_table_ready = [] {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? kPoly ^ (c >> 1) : c >> 1;
    host_table[i] = c;
  }
  return true;
}();

// a * b mod P, reflected bit order (bit 31 = x^0)
__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

// x^(8 n) mod P: square-and-multiply from x^8
__host__ __device__ inline uint32_t x8nmodp(uint64_t n) {
  uint32_t p = 1u << 31;  // x^0
  uint32_t sq = 1u << 23;  // x^8
  while (n) {
    if (n & 1) p = multmodp(sq, p);
    sq = multmodp(sq, sq);
    n >>= 1;
  }
  return p;
}

__host__ __device__ inline uint32_t crc_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
  return multmodp(x8nmodp(len2), crc1) ^ crc2;
}

constexpr int kCT = 256;

// one CTA per record: crc[i] of bytes [off[i], off[i] + len[i]) of `base`
__global__ void __launch_bounds__(kCT) crc_kernel(const unsigned char* __restrict__ base,
                                                  const uint64_t* __restrict__ off, const uint64_t* __restrict__ len,
                                                  uint32_t* __restrict__ crc) {
  __shared__ uint32_t table[256];
  __shared__ uint32_t part[kCT];
  __shared__ uint64_t plen[kCT];
  for (int i = threadIdx.x; i < 256; i += kCT) {
    uint32_t c = (uint32_t)i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? kPoly ^ (c >> 1) : c >> 1;
    table[i] = c;
  }
  __syncthreads();
  const unsigned char* p = base + off[blockIdx.x];
  const uint64_t n = len[blockIdx.x];
  const uint64_t chunk = (n + kCT - 1) / kCT;
  const uint64_t b0 = (uint64_t)threadIdx.x * chunk;
  const uint64_t b1 = b0 + chunk < n ? b0 + chunk : n;
  uint32_t c = 0xFFFFFFFFu;
  uint64_t i = b0 < n ? b0 : n;
  // 8-byte loads where aligned, bytes otherwise
  for (; i < b1 && (reinterpret_cast<uintptr_t>(p + i) & 7); ++i) c = (c >> 8) ^ table[(c ^ p[i]) & 0xffu];
  for (; i + 8 <= b1; i += 8) {
    uint64_t w = *reinterpret_cast<const uint64_t*>(p + i);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      c = (c >> 8) ^ table[(c ^ (uint32_t)w) & 0xffu];
      w >>= 8;
    }
  }
  for (; i < b1; ++i) c = (c >> 8) ^ table[(c ^ p[i]) & 0xffu];
  part[threadIdx.x] = c ^ 0xFFFFFFFFu;
  plen[threadIdx.x] = b1 > b0 ? b1 - b0 : 0;
  __syncthreads();
  // tree combine, left to right
  for (int s = 1; s < kCT; s <<= 1) {
    if ((threadIdx.x & (2 * s - 1)) == 0 && threadIdx.x + s < kCT) {
      const uint64_t l2 = plen[threadIdx.x + s];
      part[threadIdx.x] = l2 ? crc_combine(part[threadIdx.x], part[threadIdx.x + s], l2) : part[threadIdx.x];
      plen[threadIdx.x] += l2;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) crc[blockIdx.x] = n ? part[0] : 0u;
}

void put_u16(std::string& out, uint16_t v) {
  out.push_back((char)(v & 0xff));
  out.push_back((char)((v >> 8) & 0xff));
}
void put_u32(std::string& out, uint32_t v) {
  for (int i = 0; i < 4; ++i) out.push_back((char)((v >> (8 * i)) & 0xff));
}
uint32_t get_u32(const unsigned char* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

}  // namespace

uint32_t crc32_host(const void* data, uint64_t size) {
  (void)host_table_ready;
  const auto* b = static_cast<const unsigned char*>(data);
  uint32_t c = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < size; ++i) c = (c >> 8) ^ host_table[(c ^ b[i]) & 0xffu];
  return c ^ 0xFFFFFFFFu;
}

void crc32_device(const unsigned char* d_base, const std::vector<uint64_t>& off, const std::vector<uint64_t>& len,
                  uint32_t* h_crc, cudaStream_t s) {
  const size_t n = off.size();
  if (!n) return;
  DBuf<uint64_t> doff(n, s), dlen(n, s);
  DBuf<uint32_t> dcrc(n, s);
  to_device(doff.get(), off.data(), n, s);
  to_device(dlen.get(), len.data(), n, s);
  crc_kernel<<<(unsigned)n, kCT, 0, s>>>(d_base, doff.get(), dlen.get(), dcrc.get());
  RK_LAUNCH_CHECK();
  RK_CUDA_CHECK(cudaMemcpyAsync(h_crc, dcrc.get(), n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  sync(s);
}

// block_record.cpp:86-106; crc = CRC32 of the payload bytes (computed by the caller)
void write_record_file(uint32_t index, uint32_t rows, uint32_t kept, const double* payload, uint32_t crc,
                       const std::string& path) {
  std::string head;
  head.append("RNKY", 4);
  put_u16(head, 1);
  put_u32(head, index);
  put_u32(head, rows);
  put_u32(head, kept);
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(RK_RUNTIME, "cannot write " + path);
  const uint64_t count = (uint64_t)rows * kept;
  unsigned char tail[4] = {(unsigned char)(crc & 0xff), (unsigned char)((crc >> 8) & 0xff),
                           (unsigned char)((crc >> 16) & 0xff), (unsigned char)((crc >> 24) & 0xff)};
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  ok = ok && (count == 0 || std::fwrite(payload, sizeof(double), count, f) == count);  // little-endian host
  ok = ok && std::fwrite(tail, 1, 4, f) == 4;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) fail(RK_RUNTIME, "write failed for " + path);
}

// block_record.cpp:108-144, with its RecordError messages
void read_record_file(const std::string& path, uint32_t& index, uint32_t& rows, uint32_t& kept,
                      std::vector<double>& payload) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(RK_RUNTIME, "cannot open " + path);
  std::vector<unsigned char> bytes;
  unsigned char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) bytes.insert(bytes.end(), buf, buf + got);
  std::fclose(f);
  if (bytes.size() < 22) fail(RK_RECORD, "block record truncated: " + path);
  const unsigned char* p = bytes.data();
  if (std::memcmp(p, "RNKY", 4) != 0) fail(RK_RECORD, "bad block record magic in " + path);
  if ((uint16_t)(p[4] | (p[5] << 8)) != 1) fail(RK_RECORD, "unsupported block record version in " + path);
  index = get_u32(p + 6);
  rows = get_u32(p + 10);
  kept = get_u32(p + 14);
  const uint64_t count = (uint64_t)rows * kept;
  if (bytes.size() != 22 + 8 * count) fail(RK_RECORD, "block record payload truncated in " + path);
  const unsigned char* pay = p + 18;
  if (get_u32(pay + 8 * count) != crc32_host(pay, 8 * count))
    fail(RK_RECORD, "block record checksum mismatch in " + path);
  payload.resize(count);
  if (count) std::memcpy(payload.data(), pay, 8 * count);
}

}  // namespace rk
