// DEFLATE (RFC 1951) of PNG scanline streams on the device -- the compression
// step of save_slicemaps (slicemap.py:158-166), after
// ctp_png_filter_u8.  The byte stream of every image is cut into 16 KiB chunks,
// one dynamic-Huffman block per chunk, so that their concatenation (with a
// zlib header and the Adler-32 the host combines from per-chunk partials) is
// one valid zlib stream -- the pigz construction, with the whole pipeline on
// the GPU:
//   * every thread owns a 64-byte segment of the chunk, and tokens never cross
//     a segment (matches <= 64 bytes), so all per-position work is parallel;
//   * matches: for a fixed set of candidate distances (1, 2, 3, 4, the image
//     row and two rows -- the repeats that PNG-filtered slices have), the run
//     length at every position of the segment is a backward scan; the longest
//     candidate wins (ties: the shorter distance);
//   * parse: greedy within the segment, counting symbol frequencies;
//   * codes: symbols ranked by frequency in parallel, then one thread builds
//     the length-limited Huffman codes (lit/len 15, distance 15, code-length 7
//     bits) and the block header; a block that would not beat a stored block
//     is stored;
//   * bits: the 256 segments' bit lengths are prefix-summed and every thread
//     writes its tokens into a shared-memory bit buffer (atomicOr at the
//     segment seams); non-final chunks end with an empty stored block
//     (a sync flush), so every chunk is byte aligned.
// A persistent grid loops over all chunks of all images.
#include "ctp_common.cuh"

#ifndef CTP_DEFL_LBITS
#define CTP_DEFL_LBITS 1  // length-code bits charged to a match when deciding it (tuned on the c2 atlases)
#endif
#ifndef CTP_DEFL_DBITS
#define CTP_DEFL_DBITS 1  // distance-code bits charged (1 + 1: 44.2 MB; the code-length estimate 7 + 5: 46.5 MB)
#endif

namespace ctp {

constexpr int kDChunk = 16384;                  // bytes per chunk (one block)
constexpr int kDThreads = 256;
constexpr int kDSeg = kDChunk / kDThreads;      // 64: each thread scans, parses and writes its own segment
constexpr int kDOutBytes = kDChunk + 64;        // a chunk never exceeds a stored block + flush
constexpr int kDOutWords = kDOutBytes / 4;
constexpr int kDNumCand = 6;

// RFC 1951 3.2.5 length / distance tables
__constant__ uint16_t c_len_base[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                        31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dist_base[30] = {1,   2,   3,   4,   5,   7,    9,    13,   17,   25,   33,   49,   65,    97,    129,
                                         193, 257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t c_cl_order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

struct DeflateArgs {
  const uint8_t* data;        // n_streams x stream_len bytes
  int64_t stream_len;
  int32_t row_len;            // candidate distances row_len and 2 row_len
  int32_t chunks_per_stream;
  int64_t total_chunks;
  uint8_t* out;               // chunk c's bytes at out + c * kDOutBytes
  int32_t* out_bytes;         // per chunk
  unsigned long long* adler;  // per chunk: sum d_k, sum (n - k) d_k
  uint32_t* scratch;          // per CTA: kDChunk tokens
};

struct DeflateSmem {
  uint8_t buf[kDChunk];
  uint8_t best_len[kDChunk];  // matches never cross a segment: <= 64
  uint8_t best_c[kDChunk];
  uint32_t outw[kDOutWords];
  uint32_t fll[286];
  uint32_t fd[30];
  uint32_t fcl[19];
  uint8_t ll_len[286];
  uint8_t d_len[30];
  uint8_t cl_len[19];
  uint16_t ll_code[286];
  uint16_t d_code[30];
  uint16_t cl_code[19];
  uint16_t cl_sym[320];       // RLE'd code-length sequence: symbol | extra << 5
  uint16_t huf_w_sym[286];    // Huffman build work: symbols
  uint32_t huf_w[2 * 286];    // weights
  uint16_t huf_parent[2 * 286];
  uint8_t huf_depth[2 * 286];
  uint32_t warp_bits[kDThreads / 32];
  uint32_t end_bits;
  unsigned long long red[kDThreads / 32][2];
  uint32_t bhist[256];        // byte histogram of the chunk
  uint8_t litcost[256];       // estimated literal cost, quarter bits: -4 log2(p)
  uint8_t lsym_tab[259];      // match length -> length symbol - 257
  uint8_t dsym_tab[512];      // distance -> distance symbol (zlib's split table)
  uint16_t rank[286];
  int n_cl, hlit, hdist, hclen, stored;
  uint32_t header_bits;
};

// distance symbol of d in [1, 32768]: dsym_tab[d - 1] for d <= 256, else dsym_tab[256 + ((d - 1) >> 7)]
__device__ __forceinline__ int dsym_of(const DeflateSmem& S, int d) {
  return d <= 256 ? S.dsym_tab[d - 1] : S.dsym_tab[256 + ((d - 1) >> 7)];
}

__device__ __forceinline__ uint32_t bitrev(uint32_t code, int len) { return __brev(code) >> (32 - len); }

__device__ __forceinline__ void put_bits(uint32_t* w, uint32_t pos, uint32_t value, int nbits) {
  if (nbits == 0) return;
  const uint32_t word = pos >> 5, sh = pos & 31;
  atomicOr(w + word, value << sh);
  if (sh + nbits > 32) atomicOr(w + word + 1, value >> (32 - sh));
}

// The greedy parse of one segment, re-derived from shared memory by every pass
// (frequencies, bit counts, bit writing) instead of storing tokens: returns
// the token at position i (literal: value < 256; match: flag | length symbol
// | length extra | distance symbol | distance extra) and advances i.
// A match is taken only when a charged cost (CTP_DEFL_LBITS + CTP_DEFL_DBITS
// plus the extra bits) is below the estimated cost of its bytes as literals
// (-log2 of their frequency in the chunk): matches of bytes that are nearly
// free as literals are skipped, and the parse re-tries one byte later (a cheap
// form of lazy matching).
__device__ __forceinline__ uint32_t next_token(const DeflateSmem& S, const int* cand_d, int& i, int end) {
  const int L = min((int)S.best_len[i], end - i);
  if (L >= 3) {
    const int d = cand_d[S.best_c[i]];
    const int ls = S.lsym_tab[L], ds = dsym_of(S, d);
    int lit = 0;
    for (int q = 0; q < L; q++) lit += S.litcost[S.buf[i + q]];
    const int mcost = 4 * (CTP_DEFL_LBITS + c_len_extra[ls] + CTP_DEFL_DBITS + c_dist_extra[ds]);
    if (mcost >= lit) return S.buf[i++];
    i += L;
    return 0x80000000u | ((uint32_t)ls << 23) | ((uint32_t)(L - c_len_base[ls]) << 18) | ((uint32_t)ds << 13) |
           (uint32_t)(d - c_dist_base[ds]);
  }
  return S.buf[i++];
}

// rank of every used symbol in (frequency, symbol) order, all threads of the CTA
__device__ void sort_by_freq(DeflateSmem& S, const uint32_t* freq, int n) {
  for (int s = threadIdx.x; s < n; s += blockDim.x) {
    const uint32_t f = freq[s];
    if (!f) continue;
    int r = 0;
    for (int t = 0; t < n; t++) {
      const uint32_t g = freq[t];
      r += (g && (g < f || (g == f && t < s))) ? 1 : 0;
    }
    S.rank[s] = (uint16_t)r;
  }
}

// length-limited Huffman code lengths (one thread): two-queue Huffman on the
// frequency-sorted symbols; frequencies are halved until the depth fits
__device__ void huff_lengths(DeflateSmem& S, const uint32_t* freq, int n, int maxbits, uint8_t* len) {
  for (int s = 0; s < n; s++) len[s] = 0;
  int m = 0;
  for (int s = 0; s < n; s++)
    if (freq[s]) S.huf_w_sym[m++] = (uint16_t)s;
  if (m == 0) return;
  if (m == 1) {
    len[S.huf_w_sym[0]] = 1;
    return;
  }
  // symbols sorted by (frequency, symbol): ranks precomputed in parallel (sort_by_freq)
  for (int s2 = 0; s2 < n; s2++)
    if (freq[s2]) S.huf_w_sym[S.rank[s2]] = (uint16_t)s2;
  for (int shift = 0;; shift++) {
    for (int i = 0; i < m; i++) {
      const uint32_t f = freq[S.huf_w_sym[i]] >> shift;
      S.huf_w[i] = f ? f : 1;
    }
    int li = 0, ii = m, next = m;
    for (int k = 0; k < m - 1; k++) {
      int a, b;
      a = (li < m && (ii >= next || S.huf_w[li] <= S.huf_w[ii])) ? li++ : ii++;
      b = (li < m && (ii >= next || S.huf_w[li] <= S.huf_w[ii])) ? li++ : ii++;
      S.huf_w[next] = S.huf_w[a] + S.huf_w[b];
      S.huf_parent[a] = (uint16_t)next;
      S.huf_parent[b] = (uint16_t)next;
      next++;
    }
    const int root = next - 1;
    S.huf_depth[root] = 0;
    int maxd = 0;
    for (int node = root - 1; node >= 0; node--) {
      S.huf_depth[node] = S.huf_depth[S.huf_parent[node]] + 1;
      if (node < m && S.huf_depth[node] > maxd) maxd = S.huf_depth[node];
    }
    if (maxd <= maxbits) {
      for (int i = 0; i < m; i++) len[S.huf_w_sym[i]] = S.huf_depth[i];
      return;
    }
  }
}

// canonical codes (RFC 1951 3.2.2), bit-reversed for LSB-first output
__device__ void canon_codes(const uint8_t* len, int n, uint16_t* code) {
  uint16_t bl_count[16] = {0}, next_code[16];
  for (int s = 0; s < n; s++) bl_count[len[s]]++;
  bl_count[0] = 0;
  uint32_t c = 0;
  for (int b = 1; b < 16; b++) {
    c = (c + bl_count[b - 1]) << 1;
    next_code[b] = (uint16_t)c;
  }
  for (int s = 0; s < n; s++)
    code[s] = len[s] ? (uint16_t)bitrev(next_code[len[s]]++, len[s]) : 0;
}

__global__ void __launch_bounds__(kDThreads) deflate_kernel(const DeflateArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  DeflateSmem& S = *reinterpret_cast<DeflateSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cand_d[kDNumCand] = {1, 2, 3, 4, a.row_len, 2 * a.row_len};
  for (int L = tid; L < 259; L += kDThreads) {
    int sym = 0;
    if (L >= 3)
      while (sym < 28 && c_len_base[sym + 1] <= L) sym++;
    S.lsym_tab[L] = (uint8_t)sym;
  }
  for (int q = tid; q < 512; q += kDThreads) {
    const int d = q < 256 ? q + 1 : ((q - 256) << 7) + 1;  // representative distance of the entry
    int sym = 0;
    while (sym < 29 && c_dist_base[sym + 1] <= d) sym++;
    S.dsym_tab[q] = (uint8_t)sym;
  }

  for (int64_t c = blockIdx.x; c < a.total_chunks; c += gridDim.x) {
    const int64_t s = c / a.chunks_per_stream, k = c - s * a.chunks_per_stream;
    const int64_t off = k * kDChunk;
    const int n = (int)min((int64_t)kDChunk, a.stream_len - off);
    const bool last = (k == a.chunks_per_stream - 1);
    const uint8_t* src = a.data + s * a.stream_len + off;

    // ---- load, Adler-32 partials, reset
    unsigned long long s1 = 0, s2 = 0;
    for (int i = tid; i < kDChunk; i += kDThreads) {
      const uint8_t v = i < n ? __ldg(src + i) : 0;
      S.buf[i] = v;
      S.best_len[i] = 0;
      S.best_c[i] = 0;
      s1 += v;
      s2 += (unsigned long long)(n - i) * v;
    }
    for (int i = tid; i < kDOutWords; i += kDThreads) S.outw[i] = 0;
    for (int i = tid; i < 286; i += kDThreads) S.fll[i] = 0;
    if (tid < 30) S.fd[tid] = 0;
    if (tid < 19) S.fcl[tid] = 0;
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, o);
      s2 += __shfl_xor_sync(0xFFFFFFFFu, s2, o);
    }
    if (lane == 0) {
      S.red[warp][0] = s1;
      S.red[warp][1] = s2;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned long long t1 = 0, t2 = 0;
      for (int w = 0; w < kDThreads / 32; w++) {
        t1 += S.red[w][0];
        t2 += S.red[w][1];
      }
      a.adler[2 * c] = t1;
      a.adler[2 * c + 1] = t2;
    }

    // ---- literal cost estimates from the chunk's byte histogram
    for (int i = tid; i < 256; i += kDThreads) S.bhist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kDThreads) atomicAdd(&S.bhist[S.buf[i]], 1u);
    __syncthreads();
    for (int b = tid; b < 256; b += kDThreads) {
      const uint32_t h = S.bhist[b];
      const float bits = h ? __log2f((float)n / (float)h) : 15.f;
      S.litcost[b] = (uint8_t)min(60, max(1, __float2int_rn(4.f * bits)));
    }
    __syncthreads();

    // ---- matches within the own segment, then the greedy parse of it
    const int p0 = tid * kDSeg, p1 = min(n, p0 + kDSeg);
    for (int ci = 0; ci < kDNumCand; ci++) {
      const int d = cand_d[ci];
      if (d <= 0 || d > 32768 || (ci >= 4 && d <= 4) || (ci == 5 && d == cand_d[4])) continue;
      int run = 0;
      for (int i = p1 - 1; i >= p0; i--) {
        const bool eq = i >= d && S.buf[i] == S.buf[i - d];
        run = eq ? run + 1 : 0;
        if (run > S.best_len[i]) {
          S.best_len[i] = (uint8_t)run;
          S.best_c[i] = (uint8_t)ci;
        }
      }
    }
    for (int i = p0; i < p1;) {
      const uint32_t t = next_token(S, cand_d, i, p1);
      if (t & 0x80000000u) {
        atomicAdd(&S.fll[257 + ((t >> 23) & 31)], 1u);
        atomicAdd(&S.fd[(t >> 13) & 31], 1u);
      } else {
        atomicAdd(&S.fll[t], 1u);
      }
    }
    __syncthreads();

    // ---- codes and header
    if (tid == 0) {
      S.fll[256] = 1;  // end of block
      // at least two distance codes (RFC 1951 3.2.7 allows one; two keep every inflater happy)
      int nd = 0;
      for (int q = 0; q < 30; q++) nd += S.fd[q] ? 1 : 0;
      if (nd < 2) {
        if (!S.fd[0]) S.fd[0] = 1;
        else S.fd[1] = 1;
        if (nd == 0) S.fd[1] = 1;
      }
    }
    __syncthreads();
    sort_by_freq(S, S.fll, 286);
    __syncthreads();
    if (tid == 0) huff_lengths(S, S.fll, 286, 15, S.ll_len);
    __syncthreads();
    sort_by_freq(S, S.fd, 30);
    __syncthreads();
    if (tid == 0) huff_lengths(S, S.fd, 30, 15, S.d_len);
    __syncthreads();
    if (tid == 0) {
      canon_codes(S.ll_len, 286, S.ll_code);
      canon_codes(S.d_len, 30, S.d_code);
      int hlit = 286;
      while (hlit > 257 && S.ll_len[hlit - 1] == 0) hlit--;
      int hdist = 30;
      while (hdist > 1 && S.d_len[hdist - 1] == 0) hdist--;
      // run-length encode the code lengths (RFC 1951 3.2.7)
      int ncl = 0, i = 0;
      const int total = hlit + hdist;
      while (i < total) {
        const uint8_t l = i < hlit ? S.ll_len[i] : S.d_len[i - hlit];
        int run = 1;
        while (i + run < total && (i + run < hlit ? S.ll_len[i + run] : S.d_len[i + run - hlit]) == l) run++;
        i += run;
        if (l == 0) {
          while (run >= 11) {
            const int r = min(run, 138);
            S.cl_sym[ncl++] = (uint16_t)(18 | ((r - 11) << 5));
            S.fcl[18]++;
            run -= r;
          }
          if (run >= 3) {
            S.cl_sym[ncl++] = (uint16_t)(17 | ((run - 3) << 5));
            S.fcl[17]++;
            run = 0;
          }
        } else {
          S.cl_sym[ncl++] = l;
          S.fcl[l]++;
          run--;
          while (run >= 3) {
            const int r = min(run, 6);
            S.cl_sym[ncl++] = (uint16_t)(16 | ((r - 3) << 5));
            S.fcl[16]++;
            run -= r;
          }
        }
        while (run > 0) {
          S.cl_sym[ncl++] = l;
          S.fcl[l]++;
          run--;
        }
      }
      for (int q = 0; q < 19; q++) {  // ranks of the 19 code-length symbols (serial: tiny)
        if (!S.fcl[q]) continue;
        int r = 0;
        for (int t2 = 0; t2 < 19; t2++)
          r += (S.fcl[t2] && (S.fcl[t2] < S.fcl[q] || (S.fcl[t2] == S.fcl[q] && t2 < q))) ? 1 : 0;
        S.rank[q] = (uint16_t)r;
      }
      huff_lengths(S, S.fcl, 19, 7, S.cl_len);
      canon_codes(S.cl_len, 19, S.cl_code);
      int hclen = 19;
      while (hclen > 4 && S.cl_len[c_cl_order[hclen - 1]] == 0) hclen--;
      // size of the dynamic block vs a stored one
      uint64_t bits = 3 + 5 + 5 + 4 + 3 * hclen;
      for (int q = 0; q < ncl; q++) {
        const int sym = S.cl_sym[q] & 31;
        bits += S.cl_len[sym] + (sym == 16 ? 2 : sym == 17 ? 3 : sym == 18 ? 7 : 0);
      }
      for (int q = 0; q < 286; q++)
        if (S.fll[q]) bits += (uint64_t)S.fll[q] * (S.ll_len[q] + (q >= 257 ? c_len_extra[q - 257] : 0));
      for (int q = 0; q < 30; q++)
        if (S.fd[q] && (q < 30)) bits += (uint64_t)S.fd[q] * (S.d_len[q] + c_dist_extra[q]);
      // (the padding distance frequencies above add at most 2 bits: harmless)
      S.stored = bits + 16 > (uint64_t)(n + 5) * 8;
      S.n_cl = ncl;
      S.hlit = hlit;
      S.hdist = hdist;
      S.hclen = hclen;
      uint32_t pos = 0;
      if (!S.stored) {
        put_bits(S.outw, pos, last ? 1u : 0u, 1); pos += 1;
        put_bits(S.outw, pos, 2u, 2); pos += 2;  // BTYPE = 10 (dynamic)
        put_bits(S.outw, pos, (uint32_t)(hlit - 257), 5); pos += 5;
        put_bits(S.outw, pos, (uint32_t)(hdist - 1), 5); pos += 5;
        put_bits(S.outw, pos, (uint32_t)(hclen - 4), 4); pos += 4;
        for (int q = 0; q < hclen; q++) { put_bits(S.outw, pos, S.cl_len[c_cl_order[q]], 3); pos += 3; }
        for (int q = 0; q < ncl; q++) {
          const int sym = S.cl_sym[q] & 31, ex = S.cl_sym[q] >> 5;
          put_bits(S.outw, pos, S.cl_code[sym], S.cl_len[sym]); pos += S.cl_len[sym];
          const int eb = sym == 16 ? 2 : sym == 17 ? 3 : sym == 18 ? 7 : 0;
          put_bits(S.outw, pos, (uint32_t)ex, eb); pos += eb;
        }
      }
      S.header_bits = pos;
    }
    __syncthreads();

    int nbytes;
    if (S.stored) {
      // stored block: header bits, byte align, LEN, NLEN, the raw bytes (RFC 1951 3.2.4)
      if (tid == 0) {
        put_bits(S.outw, 0, last ? 1u : 0u, 3);  // BFINAL, BTYPE = 00
        uint8_t* ob = reinterpret_cast<uint8_t*>(S.outw);
        ob[1] = (uint8_t)(n & 0xFF);
        ob[2] = (uint8_t)(n >> 8);
        ob[3] = (uint8_t)(~n & 0xFF);
        ob[4] = (uint8_t)((~n >> 8) & 0xFF);
      }
      __syncthreads();
      uint8_t* ob = reinterpret_cast<uint8_t*>(S.outw);
      for (int i = tid; i < n; i += kDThreads) ob[5 + i] = S.buf[i];
      nbytes = 5 + n;
    } else {
      // token bits: thread t's segment after the header and segments 0..t-1
      uint32_t b = 0;
      for (int i = p0; i < p1;) {
        const uint32_t t = next_token(S, cand_d, i, p1);
        if (t & 0x80000000u) {
          const int ls = (t >> 23) & 31, ds = (t >> 13) & 31;
          b += S.ll_len[257 + ls] + c_len_extra[ls] + S.d_len[ds] + c_dist_extra[ds];
        } else {
          b += S.ll_len[t];
        }
      }
      uint32_t incl = b;  // block-wide exclusive scan of the segments' bit counts
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) S.warp_bits[warp] = incl;
      __syncthreads();
      uint32_t before = 0;
      for (int w = 0; w < warp; w++) before += S.warp_bits[w];
      uint32_t pos = S.header_bits + before + incl - b;
      for (int i = p0; i < p1;) {
        const uint32_t t = next_token(S, cand_d, i, p1);
        if (t & 0x80000000u) {
          const int ls = (t >> 23) & 31, ds = (t >> 13) & 31;
          put_bits(S.outw, pos, S.ll_code[257 + ls], S.ll_len[257 + ls]); pos += S.ll_len[257 + ls];
          put_bits(S.outw, pos, (t >> 18) & 31u, c_len_extra[ls]); pos += c_len_extra[ls];
          put_bits(S.outw, pos, S.d_code[ds], S.d_len[ds]); pos += S.d_len[ds];
          put_bits(S.outw, pos, t & 0x1FFFu, c_dist_extra[ds]); pos += c_dist_extra[ds];
        } else {
          put_bits(S.outw, pos, S.ll_code[t], S.ll_len[t]); pos += S.ll_len[t];
        }
      }
      if (tid == kDThreads - 1) S.end_bits = pos;  // end of the last segment
      __syncthreads();
      pos = S.end_bits;
      if (tid == 0) put_bits(S.outw, pos, S.ll_code[256], S.ll_len[256]);  // end of block
      pos += S.ll_len[256];
      if (!last) {  // sync flush: an empty stored block, byte aligned
        pos += 3;
        pos = (pos + 7) & ~7u;
        if (tid == 0) {
          uint8_t* ob = reinterpret_cast<uint8_t*>(S.outw);
          ob[pos / 8 + 0] = 0x00;
          ob[pos / 8 + 1] = 0x00;
          ob[pos / 8 + 2] = 0xFF;
          ob[pos / 8 + 3] = 0xFF;
        }
        nbytes = pos / 8 + 4;
      } else {
        nbytes = (pos + 7) / 8;
      }
      __syncthreads();
    }
    // stored blocks already end byte aligned; a non-final one needs no flush
    uint8_t* dst = a.out + c * (int64_t)kDOutBytes;
    const uint8_t* ob = reinterpret_cast<const uint8_t*>(S.outw);
    for (int i = tid; i < nbytes; i += kDThreads) dst[i] = ob[i];
    if (tid == 0) a.out_bytes[c] = nbytes;
    __syncthreads();
  }
}

// gather the chunks' bytes into one contiguous buffer (offsets: exclusive scan of the sizes)
__global__ void __launch_bounds__(256) deflate_compact_kernel(const uint8_t* __restrict__ out,
                                                              const int32_t* __restrict__ sizes,
                                                              const int64_t* __restrict__ offsets,
                                                              uint8_t* __restrict__ dst) {
  const int64_t c = blockIdx.x;
  const uint8_t* src = out + c * (int64_t)kDOutBytes;
  uint8_t* d = dst + offsets[c];
  const int n = sizes[c];
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = src[i];
}

}  // namespace ctp

using namespace ctp;

extern "C" {

int ctp_deflate_geometry(int32_t* chunk_bytes, int32_t* chunk_out_bytes) {
  CTP_REQUIRE(chunk_bytes && chunk_out_bytes, CTP_E_INVALID, "ctp_deflate_geometry: null pointer");
  *chunk_bytes = kDChunk;
  *chunk_out_bytes = kDOutBytes;
  return CTP_OK;
}

int ctp_deflate_u8(const uint8_t* data, int64_t n_streams, int64_t stream_len, int32_t row_len, uint8_t* out,
                   int32_t* out_bytes, uint64_t* adler, uint32_t* scratch, int32_t grid, void* stream) {
  CTP_REQUIRE(data && out && out_bytes && adler && scratch, CTP_E_INVALID, "ctp_deflate_u8: null pointer");
  CTP_REQUIRE(n_streams >= 1 && stream_len >= 1 && grid >= 1, CTP_E_INVALID, "ctp_deflate_u8: bad sizes");
  DeflateArgs a;
  a.data = data;
  a.stream_len = stream_len;
  a.row_len = row_len;
  a.chunks_per_stream = (int32_t)((stream_len + kDChunk - 1) / kDChunk);
  a.total_chunks = n_streams * a.chunks_per_stream;
  a.out = out;
  a.out_bytes = out_bytes;
  a.adler = reinterpret_cast<unsigned long long*>(adler);
  a.scratch = scratch;
  const size_t sm = sizeof(DeflateSmem);
  CTP_CUDA_CALL(cudaFuncSetAttribute(deflate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int64_t g = grid;
  if (g > a.total_chunks) g = a.total_chunks;
  deflate_kernel<<<(unsigned)g, kDThreads, sm, as_stream(stream)>>>(a);
  CTP_CUDA_CHECK_LAUNCH("deflate_kernel");
  return CTP_OK;
}

int ctp_deflate_compact(const uint8_t* out, const int32_t* out_bytes, const int64_t* offsets, int64_t total_chunks,
                        uint8_t* dst, void* stream) {
  CTP_REQUIRE(out && out_bytes && offsets && dst, CTP_E_INVALID, "ctp_deflate_compact: null pointer");
  CTP_REQUIRE(total_chunks >= 1 && total_chunks < (1LL << 31), CTP_E_INVALID, "ctp_deflate_compact: bad count");
  deflate_compact_kernel<<<(unsigned)total_chunks, 256, 0, as_stream(stream)>>>(out, out_bytes, offsets, dst);
  CTP_CUDA_CHECK_LAUNCH("deflate_compact_kernel");
  return CTP_OK;
}

}  // extern "C"
