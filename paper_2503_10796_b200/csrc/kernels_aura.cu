// kernels_aura.cu -- delta-encoded + LZ4-compressed aura messages.
//
// Sec. "Data Transfer Minimization": sender and receiver hold the same
// reference; the sender reorders the message to the reference (placeholders for agents
// that left, new agents appended), writes the difference against the reference and
// compresses it with LZ4 (evaluation P:6911-6937).  Readings R46-R51:
//   R46 reference = an aura message in ascending id order (bdm_aura_reference);
//   R47 slot r < nref carries the message agent with id ref.id[r] or a placeholder
//       (presence bit 0); new agents follow at nref.. in message order;
//   R48 difference = XOR of the IEEE bit patterns of x, y, z, d and of flags;
//   R49 payload = presence words | x, y, z, d columns as 8 byte planes each | flags as
//       4 byte planes | ids of the new agents;
//   R50 LZ4 block format over independent 1024-byte chunks, greedy parse with an
//       11-bit hash bucket per 4-byte sequence;
//   R51 decoding returns the reference-order survivors, then the new agents.
//
//   k_aura_match     binary search of every message id in the reference; presence bits
//   scan             rank of the new agents
//   k_aura_fill      XOR / raw values into the byte planes
//   k_lz4_compress   one warp per 1 KB chunk in shared memory: bucket candidates of all
//                    positions (match_any), then the greedy parse 32 positions per probe
//   scan + k_aura_pack   header, chunk sizes, chunks concatenated
//   k_lz4_decompress / k_aura_unfill   the inverse
// Byte planes make the XOR deltas of slowly moving agents LZ4-friendly: their high
// bytes are zero and land in long zero runs (the paper compresses its object buffers
// as they are).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "bdm_internal.cuh"

namespace bdm {

constexpr int kChunk = 1024;                       // payload bytes per LZ4 block
constexpr int kChunkCap = kChunk + kChunk / 255 + 16;  // worst-case block size
constexpr int kHBits = 11;
constexpr uint32_t kMagic = 0x31414442u;           // "BDA1"
constexpr int kHdr = 40;

struct AuraHeader {
    uint32_t magic, chunk;
    uint64_t nref, nnew, size;
    uint32_t nch, zero;
};
static_assert(sizeof(AuraHeader) == kHdr, "header layout");

static int64_t payload_size(int64_t nref, int64_t nnew) {
    const int64_t ns = nref + nnew;
    return 4 * ((nref + 31) / 32) + 32 * ns + 4 * ns + 4 * nnew;
}

// ------------------------------------------------------------------ encode
__global__ void k_aura_match(int64_t n, const uint32_t *__restrict__ id,
                             const uint32_t *__restrict__ rid, int64_t nref,
                             uint32_t *__restrict__ slot, uint32_t *__restrict__ isnew,
                             uint32_t *__restrict__ pres, uint32_t *__restrict__ inv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0) isnew[n] = 0u;
    if (i >= n) return;
    const uint32_t me = id[i];
    int64_t lo = 0, hi = nref;
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (rid[mid] < me) lo = mid + 1; else hi = mid;
    }
    const bool found = lo < nref && rid[lo] == me;
    slot[i] = found ? (uint32_t)lo : 0xFFFFFFFFu;
    isnew[i] = found ? 0u : 1u;
    if (found) {
        atomicOr(&pres[lo >> 5], 1u << (lo & 31));
        inv[lo] = (uint32_t)i;  // reference slot -> message index
    }
}

// message index of each new agent, by its rank
__global__ void k_aura_newlist(int64_t n, const uint32_t *__restrict__ slot,
                               const uint32_t *__restrict__ newrank, uint32_t *__restrict__ newlist) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && slot[i] == 0xFFFFFFFFu) newlist[newrank[i]] = (uint32_t)i;
}

struct AuraView {
    const double *x, *y, *z, *d;
    const uint32_t *id, *flags;
};

// One thread per payload slot (coalesced byte-plane writes); nnew is read on the device.
__global__ void k_aura_fill(int64_t n, AuraView m, AuraView r, int64_t nref,
                            const uint32_t *__restrict__ inv, const uint32_t *__restrict__ newlist,
                            const uint32_t *__restrict__ newrank, uint8_t *__restrict__ pay) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nnew = (int64_t)newrank[n];
    const int64_t ns = nref + nnew, nw = (nref + 31) / 32;
    if (s >= ns) return;
    const bool matched = s < nref;
    const uint32_t i = matched ? inv[s] : newlist[s - nref];
    if (i == 0xFFFFFFFFu) return;  // placeholder: zeros
    unsigned long long v[4] = {
        (unsigned long long)__double_as_longlong(m.x[i]), (unsigned long long)__double_as_longlong(m.y[i]),
        (unsigned long long)__double_as_longlong(m.z[i]), (unsigned long long)__double_as_longlong(m.d[i])};
    uint32_t f = m.flags[i];
    if (matched) {
        v[0] ^= (unsigned long long)__double_as_longlong(r.x[s]);
        v[1] ^= (unsigned long long)__double_as_longlong(r.y[s]);
        v[2] ^= (unsigned long long)__double_as_longlong(r.z[s]);
        v[3] ^= (unsigned long long)__double_as_longlong(r.d[s]);
        f ^= r.flags[s];
    } else {
        uint8_t *nid = pay + 4 * nw + 36 * ns + 4 * (s - nref);
        const uint32_t me = m.id[i];
#pragma unroll
        for (int b = 0; b < 4; ++b) nid[b] = (uint8_t)(me >> (8 * b));
    }
    uint8_t *col = pay + 4 * nw;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int b = 0; b < 8; ++b) col[(int64_t)(8 * c + b) * ns + s] = (uint8_t)(v[c] >> (8 * b));
    uint8_t *fcol = col + 32 * ns;
#pragma unroll
    for (int b = 0; b < 4; ++b) fcol[(int64_t)b * ns + s] = (uint8_t)(f >> (8 * b));
}

// ---- LZ4 (R50), one warp per 1 KB chunk staged in shared memory
struct LzWarp {
    uint8_t src[kChunk + 16];
    uint16_t cand[kChunk];
    uint16_t table[1 << kHBits];
};
constexpr int kLzWarps = 8;

__device__ __forceinline__ uint32_t rd32s(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

__device__ __forceinline__ int len_bytes(int L) { return L >= 15 ? (L - 15) / 255 + 1 : 0; }

// Writes the 255-run length code of L >= 15 at dst[o..] (one lane).
__device__ __forceinline__ void put_len(uint8_t *dst, int o, int L) {
    L -= 15;
    while (L >= 255) {
        dst[o++] = 255;
        L -= 255;
    }
    dst[o] = (uint8_t)L;
}

// One sequence (literals src[a, a + nlit), then a match of mlen at distance off if
// mlen > 0), written by the whole warp; returns the new output position.
__device__ __forceinline__ int warp_sequence(const uint8_t *src, int a, int nlit, int off, int mlen,
                                             uint8_t *__restrict__ dst, int o, int lane) {
    const int lb = len_bytes(nlit);
    const int olit = o + 1 + lb;
    for (int k = lane; k < nlit; k += 32) dst[olit + k] = src[a + k];
    int e = olit + nlit;
    if (lane == 0) {
        uint8_t t = (uint8_t)((nlit < 15 ? nlit : 15) << 4);
        if (nlit >= 15) put_len(dst, o + 1, nlit);
        if (mlen > 0) {
            dst[e] = (uint8_t)(off & 255);
            dst[e + 1] = (uint8_t)(off >> 8);
            const int mm = mlen - 4;
            t |= (uint8_t)(mm < 15 ? mm : 15);
            if (mm >= 15) put_len(dst, e + 2, mm);
        }
        dst[o] = t;
    }
    if (mlen > 0) e += 2 + len_bytes(mlen - 4);
    return e;
}

__device__ __forceinline__ int64_t dev_payload_size(int64_t nref, int64_t nnew) {
    const int64_t ns = nref + nnew;
    return 4 * ((nref + 31) / 32) + 32 * ns + 4 * ns + 4 * nnew;
}

// The payload size follows from nnew = newrank[n] on the device; chunks past it
// report size 0 (the grid covers the bound for nnew = n).
__global__ void __launch_bounds__(32 * kLzWarps) k_lz4_compress(const uint8_t *__restrict__ pay,
                                                               const uint32_t *__restrict__ newrank,
                                                               int64_t nmsg, int64_t nref,
                                                               int64_t nch_max,
                                                               uint8_t *__restrict__ tmp,
                                                               uint32_t *__restrict__ csize) {
    extern __shared__ __align__(16) unsigned char lz_smem[];
    LzWarp &S = reinterpret_cast<LzWarp *>(lz_smem)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int64_t c = blockIdx.x * (int64_t)kLzWarps + (threadIdx.x >> 5);
    if (c >= nch_max) return;
    const int64_t size = dev_payload_size(nref, (int64_t)newrank[nmsg]);
    const int64_t nch = (size + kChunk - 1) / kChunk;
    if (c >= nch) {
        if (lane == 0) csize[c] = 0u;
        return;
    }
    const int n = (int)(size - c * kChunk < kChunk ? size - c * kChunk : kChunk);
    const uint8_t *g = pay + c * kChunk;
    if (n == kChunk) {
        const uint4 *g4 = reinterpret_cast<const uint4 *>(g);
        for (int k = lane; k < kChunk / 16; k += 32) reinterpret_cast<uint4 *>(S.src)[k] = g4[k];
    } else {
        for (int k = lane; k < n; k += 32) S.src[k] = g[k];
    }
    for (int k = lane; k < (1 << kHBits); k += 32) S.table[k] = 0xFFFFu;
    __syncwarp();
    // pass 1: candidate of every position = last earlier position in the same bucket
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < n; base += 32) {
        const int p = base + lane;
        const bool valid = p + 4 <= n;
        const uint32_t h = valid ? (rd32s(S.src + p) * 2654435761u) >> (32 - kHBits)
                                 : (1u << kHBits) + (uint32_t)lane;
        const unsigned grp = __match_any_sync(0xffffffffu, h);
        const unsigned before = grp & lt;
        uint16_t cd = 0xFFFFu;
        if (valid) cd = before ? (uint16_t)(base + 31 - __clz(before)) : S.table[h];
        if (p < n) S.cand[p] = cd;
        __syncwarp();
        if (valid && !(grp & ~(lt | (1u << lane)))) S.table[h] = (uint16_t)p;  // last of its group
        __syncwarp();
    }
    // pass 2: greedy parse, 32 positions per probe
    uint8_t *dst = tmp + c * kChunkCap;
    const int limit = n - 12;
    int ip = 0, anchor = 0, o = 0;
    while (ip < limit) {
        const int p = ip + lane;
        bool ok = false;
        if (p < limit) {
            const uint16_t r = S.cand[p];
            ok = r != 0xFFFFu && rd32s(S.src + r) == rd32s(S.src + p);
        }
        const unsigned b = __ballot_sync(0xffffffffu, ok);
        if (!b) {
            ip = min(ip + 32, limit);
            continue;
        }
        ip += __ffs(b) - 1;
        const int ref = S.cand[ip];
        int len = 4;
        for (;;) {
            const int q = ip + len + lane;
            const bool eq = q < n - 5 && S.src[ref + len + lane] == S.src[q];
            const unsigned mb = __ballot_sync(0xffffffffu, !eq);
            if (mb) {
                len += __ffs(mb) - 1;
                break;
            }
            len += 32;
        }
        o = warp_sequence(S.src, anchor, ip - anchor, ip - ref, len, dst, o, lane);
        ip += len;
        anchor = ip;
    }
    o = warp_sequence(S.src, anchor, n - anchor, 0, 0, dst, o, lane);
    if (lane == 0) csize[c] = (uint32_t)o;
}

// Header, chunk sizes, chunks (a warp per chunk).  off holds the exclusive scan of the
// chunk sizes over nch_max + 1 entries (chunks past nch have size 0).  Writes nothing
// if the stream does not fit in out_cap; res = {stream bytes, fits}.
__global__ void k_aura_pack(const uint8_t *__restrict__ tmp, const uint32_t *__restrict__ off,
                            const uint32_t *__restrict__ newrank, int64_t n, int64_t nref,
                            int64_t nch_max, int64_t out_cap, uint8_t *__restrict__ out,
                            long long *__restrict__ res) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nnew = (int64_t)newrank[n], size = dev_payload_size(nref, nnew);
    const int64_t nch = (size + kChunk - 1) / kChunk;
    const int64_t bytes = kHdr + 4 * nch + (int64_t)off[nch_max];
    const bool fits = bytes <= out_cap;
    if (w == 0 && lane == 0) {
        res[0] = bytes;
        res[1] = fits ? 1 : 0;
        if (fits) {
            AuraHeader h{kMagic, (uint32_t)kChunk, (uint64_t)nref, (uint64_t)nnew, (uint64_t)size,
                         (uint32_t)nch, 0u};
            memcpy(out, &h, sizeof(h));
        }
    }
    if (!fits || w >= nch) return;
    const uint32_t a = off[w], k = off[w + 1] - a;
    if (lane == 0) memcpy(out + kHdr + 4 * w, &k, 4);
    const uint8_t *s = tmp + w * kChunkCap;
    uint8_t *d = out + kHdr + 4 * nch + a;
    for (uint32_t j = lane; j < k; j += 32) d[j] = s[j];
}

// ------------------------------------------------------------------ decode
__global__ void __launch_bounds__(32 * kLzWarps) k_lz4_decompress(const uint8_t *__restrict__ in,
                                                                 const uint32_t *__restrict__ off,
                                                                 const uint32_t *__restrict__ len,
                                                                 int64_t size, int64_t nch,
                                                                 uint8_t *__restrict__ pay,
                                                                 int *__restrict__ err) {
    __shared__ __align__(16) uint8_t outb[kLzWarps][kChunk];
    __shared__ __align__(16) uint8_t inb[kLzWarps][kChunkCap + 16];
    const int lane = threadIdx.x & 31;
    const int64_t c = blockIdx.x * (int64_t)kLzWarps + (threadIdx.x >> 5);
    if (c >= nch) return;
    uint8_t *dst = outb[threadIdx.x >> 5];
    const int n = (int)len[c];
    const int cap = (int)(size - c * kChunk < kChunk ? size - c * kChunk : kChunk);
    // the parse is a chain of dependent byte reads: stage the block in shared memory
    // (a block longer than any this encoder writes is parsed from global memory)
    const uint8_t *gsrc = in + off[c];
    const uint8_t *src = gsrc;
    if (n <= kChunkCap + 16) {
        uint8_t *st = inb[threadIdx.x >> 5];
        for (int k = lane; k < n; k += 32) st[k] = gsrc[k];
        __syncwarp();
        src = st;
    }
    int i = 0, o = 0;
    bool bad = false;
    while (i < n) {  // warp-uniform parse; copies are lane-parallel
        const uint8_t t = src[i++];
        int nlit = t >> 4;
        if (nlit == 15) {
            uint8_t b;
            do {
                if (i >= n) { bad = true; break; }
                b = src[i++];
                nlit += b;
            } while (b == 255);
            if (bad) break;
        }
        if (i + nlit > n || o + nlit > cap) { bad = true; break; }
        for (int k = lane; k < nlit; k += 32) dst[o + k] = src[i + k];
        i += nlit;
        o += nlit;
        if (i == n) break;
        if (i + 2 > n) { bad = true; break; }
        const int ofs = (int)src[i] | ((int)src[i + 1] << 8);
        i += 2;
        int mlen = (t & 15) + 4;
        if ((t & 15) == 15) {
            uint8_t b;
            do {
                if (i >= n) { bad = true; break; }
                b = src[i++];
                mlen += b;
            } while (b == 255);
            if (bad) break;
        }
        if (ofs == 0 || ofs > o || o + mlen > cap) { bad = true; break; }
        __syncwarp();
        const int step = ofs < 32 ? ofs : 32;  // overlapping copies in rounds of ofs bytes
        for (int d0 = 0; d0 < mlen; d0 += step) {
            if (lane < step && d0 + lane < mlen) dst[o + d0 + lane] = dst[o + d0 + lane - ofs];
            __syncwarp();
        }
        o += mlen;
    }
    __syncwarp();
    if (bad || o != cap) {
        if (lane == 0) atomicExch(err, 1);
        return;
    }
    uint8_t *g = pay + c * kChunk;
    if (cap == kChunk) {
        for (int k = lane; k < kChunk / 16; k += 32)
            reinterpret_cast<uint4 *>(g)[k] = reinterpret_cast<const uint4 *>(dst)[k];
    } else {
        for (int k = lane; k < cap; k += 32) g[k] = dst[k];
    }
}

__global__ void k_aura_presence_counts(const uint8_t *__restrict__ pay, int64_t nw,
                                       uint32_t *__restrict__ cnt) {
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w == 0) cnt[nw] = 0u;
    if (w >= nw) return;
    uint32_t v;
    memcpy(&v, pay + 4 * w, 4);
    cnt[w] = (uint32_t)__popc(v);
}

struct AuraOut {
    double *x, *y, *z, *d;
    uint32_t *id, *flags;
};

__global__ void k_aura_unfill(const uint8_t *__restrict__ pay, int64_t nref, int64_t nnew,
                              const uint32_t *__restrict__ wprefix, AuraView r, AuraOut o) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t ns = nref + nnew, nw = (nref + 31) / 32;
    if (s >= ns) return;
    int64_t dst;
    if (s < nref) {
        uint32_t word;
        memcpy(&word, pay + 4 * (s >> 5), 4);
        if (!((word >> (s & 31)) & 1u)) return;  // placeholder
        dst = (int64_t)wprefix[s >> 5] + __popc(word & ((1u << (s & 31)) - 1u));
    } else {
        dst = (int64_t)wprefix[nw] + (s - nref);
    }
    const uint8_t *col = pay + 4 * nw;
    unsigned long long v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        unsigned long long a = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) a |= (unsigned long long)col[(int64_t)(8 * c + b) * ns + s] << (8 * b);
        v[c] = a;
    }
    const uint8_t *fcol = col + 32 * ns;
    uint32_t f = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) f |= (uint32_t)fcol[(int64_t)b * ns + s] << (8 * b);
    uint32_t me;
    if (s < nref) {
        v[0] ^= (unsigned long long)__double_as_longlong(r.x[s]);
        v[1] ^= (unsigned long long)__double_as_longlong(r.y[s]);
        v[2] ^= (unsigned long long)__double_as_longlong(r.z[s]);
        v[3] ^= (unsigned long long)__double_as_longlong(r.d[s]);
        f ^= r.flags[s];
        me = r.id[s];
    } else {
        const uint8_t *nid = fcol + 4 * ns + 4 * (s - nref);
        me = (uint32_t)nid[0] | ((uint32_t)nid[1] << 8) | ((uint32_t)nid[2] << 16) |
             ((uint32_t)nid[3] << 24);
    }
    o.x[dst] = __longlong_as_double((long long)v[0]);
    o.y[dst] = __longlong_as_double((long long)v[1]);
    o.z[dst] = __longlong_as_double((long long)v[2]);
    o.d[dst] = __longlong_as_double((long long)v[3]);
    o.id[dst] = me;
    o.flags[dst] = f;
}

// ------------------------------------------------------------------ reference (R46)
// ------------------------------------------------------------------ radix sort by id
// The reference order of a message (ascending id) as a least-significant-
// digit radix sort of (id, index) pairs: four stable passes over 8-bit digits.  A block
// owns a tile of kRsTile consecutive pairs.  k_rs_hist counts its digits into
// hist[digit * nblocks + block]; the exclusive scan of that table (digit-major) is each
// block's first output slot per digit; k_rs_scatter ranks the tile's pairs stably (round
// by round of 256 consecutive pairs: earlier rounds, earlier warps, lower lanes with the
// same digit, found with match.any) and moves them.  Ids are unique, so the result does
// not depend on stability between equal keys, only between equal digits.
constexpr int kRsThreads = 256;
constexpr int kRsRounds = 8;
constexpr int kRsTile = kRsThreads * kRsRounds;

__global__ void __launch_bounds__(kRsThreads) k_rs_hist(int64_t n, const uint32_t *__restrict__ key,
                                                        int shift, uint32_t *__restrict__ hist,
                                                        int64_t nblocks) {
    __shared__ uint32_t cnt[256];
    cnt[threadIdx.x] = 0u;
    __syncthreads();
    const int64_t base = blockIdx.x * (int64_t)kRsTile;
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r) {
        const int64_t i = base + r * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&cnt[(key[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
    if (blockIdx.x == 0 && threadIdx.x == 0) hist[256 * nblocks] = 0u;
}

__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(
    int64_t n, const uint32_t *__restrict__ key, const uint32_t *__restrict__ val /* NULL: index */,
    int shift, const uint32_t *__restrict__ offs, int64_t nblocks, uint32_t *__restrict__ key_out,
    uint32_t *__restrict__ val_out) {
    __shared__ uint32_t wcnt[kRsThreads / 32][256];
    __shared__ uint32_t running[256];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    running[t] = offs[t * nblocks + blockIdx.x];
    const int64_t base = blockIdx.x * (int64_t)kRsTile;
    for (int r = 0; r < kRsRounds; ++r) {
#pragma unroll
        for (int q = 0; q < kRsThreads / 32; ++q) wcnt[q][t] = 0u;
        __syncthreads();  // (also orders the previous round's update of `running`)
        const int64_t i = base + r * kRsThreads + t;
        const bool on = i < n;
        const uint32_t k = on ? key[i] : 0u;
        const uint32_t d = on ? (k >> shift) & 255u : 256u + (uint32_t)lane;  // idle lanes match nobody
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t below = __popc(peers & ((1u << lane) - 1u));
        if (on && below == 0u) wcnt[w][d] = __popc(peers);
        __syncthreads();
        if (on) {
            uint32_t pos = running[d] + below;
            for (int q = 0; q < w; ++q) pos += wcnt[q][d];
            key_out[pos] = k;
            val_out[pos] = val ? val[i] : (uint32_t)i;
        }
        __syncthreads();
        uint32_t tot = 0;
#pragma unroll
        for (int q = 0; q < kRsThreads / 32; ++q) tot += wcnt[q][t];
        running[t] += tot;
    }
}

__global__ void k_aura_gather(int64_t n, const uint32_t *__restrict__ perm, AuraView m, AuraOut o,
                              const uint32_t *__restrict__ sorted_id) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = perm[i];
    o.x[i] = m.x[p];
    o.y[i] = m.y[p];
    o.z[i] = m.z[p];
    o.d[i] = m.d[p];
    o.id[i] = sorted_id[i];
    o.flags[i] = m.flags[p];
}

// ------------------------------------------------------------------ workspace
template <class T>
static bdm_status ensure(T **p, int64_t &cap, int64_t need) {
    if (need <= cap && *p) return BDM_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    cap = 0;
    const int64_t n = need + need / 4 + 256;
    BDM_CUDA_TRY(cudaMalloc((void **)p, (size_t)n * sizeof(T)));
    cap = n;
    return BDM_OK;
}

static bdm_status ensure_scan(Ctx *c, int64_t m) {
    const int64_t nb = scan_block_count(m) + 1;
    if (nb <= c->block_sums_cap) return BDM_OK;
    BDM_CUDA_TRY(cudaDeviceSynchronize());
    ctx_free(c, c->block_sums);  // (allocated through the context's allocator, bdm_create_ex)
    c->block_sums = nullptr;
    c->block_sums_cap = 0;
    BDM_CUDA_TRY(ctx_malloc(c, (void **)&c->block_sums, (size_t)nb * sizeof(uint32_t)));
    c->block_sums_cap = nb;
    return BDM_OK;
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

static AuraView view(const bdm_agents *a) {
    return AuraView{a->x, a->y, a->z, a->diameter, a->id, a->flags};
}
static AuraOut outv(bdm_agents *a) {
    return AuraOut{a->x, a->y, a->z, a->diameter, a->id, a->flags};
}

int64_t aura_max_size(int64_t nref, int64_t n) {
    const int64_t size = payload_size(nref, n);
    const int64_t nch = (size + kChunk - 1) / kChunk;
    return kHdr + 4 * nch + nch * (int64_t)kChunkCap;
}

bdm_status launch_aura_reference(Ctx *c, const bdm_agents *m, bdm_agents *r, cudaStream_t st) {
    const int64_t n = m->n;
    AuraWs &W = c->aura;
    bdm_status s;
    if ((s = ensure(&W.u32a, W.u32a_cap, 2 * n + 2)) != BDM_OK) return s;
    if ((s = ensure(&W.u32b, W.u32b_cap, 2 * n + 2)) != BDM_OK) return s;
    uint32_t *const kb[2] = {W.u32a, W.u32a + n + 1}, *const vb[2] = {W.u32b, W.u32b + n + 1};
    uint32_t *keys_out = kb[1], *vals_out = vb[1];  // four passes end in buffer 1
    if (n > 0) {
        const int64_t nb = (n + kRsTile - 1) / kRsTile;
        if ((s = ensure(&W.tmp, W.tmp_cap, (256 * nb + 1) * (int64_t)sizeof(uint32_t))) != BDM_OK) return s;
        if ((s = ensure_scan(c, 256 * nb + 1)) != BDM_OK) return s;
        uint32_t *const hist = reinterpret_cast<uint32_t *>(W.tmp);
        for (int pass = 0; pass < 4; ++pass) {
            const uint32_t *kin = pass == 0 ? m->id : kb[(pass + 1) & 1];
            const uint32_t *vin = pass == 0 ? nullptr : vb[(pass + 1) & 1];
            k_rs_hist<<<(unsigned)nb, kRsThreads, 0, st>>>(n, kin, 8 * pass, hist, nb);
            if ((s = launch_scan_u32(c, hist, 256 * nb + 1, st)) != BDM_OK) return s;
            k_rs_scatter<<<(unsigned)nb, kRsThreads, 0, st>>>(n, kin, vin, 8 * pass, hist, nb,
                                                              kb[pass & 1], vb[pass & 1]);
            c->launches += 2;
        }
        k_aura_gather<<<nblk(n, 256), 256, 0, st>>>(n, vals_out, view(m), outv(r), keys_out);
        c->launches += 1;
        BDM_LAUNCH_CHECK("aura reference");
    }
    r->n = n;
    return BDM_OK;
}

bdm_status launch_aura_encode(Ctx *c, const bdm_agents *m, const bdm_agents *r, uint8_t *out,
                              int64_t out_cap, int64_t *out_size, cudaStream_t st) {
    // one synchronization: every size past the match is read on the device, the grids
    // cover the bound nnew = n
    const int64_t n = m->n, nref = r->n;
    AuraWs &W = c->aura;
    bdm_status s;
    if ((s = ensure(&W.u32a, W.u32a_cap, (n + 1) + nref + n + 1)) != BDM_OK) return s;
    if ((s = ensure(&W.u32b, W.u32b_cap, n + 1)) != BDM_OK) return s;
    uint32_t *slot = W.u32a, *inv = W.u32a + n + 1, *newlist = inv + nref, *newrank = W.u32b;
    const int64_t pmax = payload_size(nref, n);
    const int64_t nch_max = (pmax + kChunk - 1) / kChunk;
    if ((s = ensure(&W.pay, W.pay_cap, pmax)) != BDM_OK) return s;
    if ((s = ensure(&W.tmp, W.tmp_cap, nch_max * (int64_t)kChunkCap)) != BDM_OK) return s;
    if ((s = ensure(&W.sizes, W.sizes_cap, nch_max + 1)) != BDM_OK) return s;
    if ((s = ensure_scan(c, (n > nch_max ? n : nch_max) + 1)) != BDM_OK) return s;
    if (!W.res) BDM_CUDA_TRY(cudaMalloc(&W.res, 2 * sizeof(long long)));
    BDM_CUDA_TRY(cudaMemsetAsync(W.pay, 0, (size_t)pmax, st));
    if (nref > 0) BDM_CUDA_TRY(cudaMemsetAsync(inv, 0xFF, (size_t)nref * 4, st));
    BDM_CUDA_TRY(cudaMemsetAsync(W.sizes + nch_max, 0, sizeof(uint32_t), st));
    if (n > 0) {
        k_aura_match<<<nblk(n, 256), 256, 0, st>>>(n, m->id, r->id, nref, slot, newrank,
                                                    (uint32_t *)W.pay, inv);
        c->launches += 1;
    } else {
        BDM_CUDA_TRY(cudaMemsetAsync(newrank, 0, sizeof(uint32_t), st));
    }
    BDM_LAUNCH_CHECK("k_aura_match");
    if ((s = launch_scan_u32(c, newrank, n + 1, st)) != BDM_OK) return s;
    if (n > 0) {
        k_aura_newlist<<<nblk(n, 256), 256, 0, st>>>(n, slot, newrank, newlist);
        c->launches += 1;
    }
    if (nref + n > 0) {
        // the presence words were written in place; the planes start after them
        k_aura_fill<<<nblk(nref + n, 256), 256, 0, st>>>(n, view(m), view(r), nref, inv, newlist,
                                                         newrank, W.pay);
        c->launches += 1;
    }
    BDM_LAUNCH_CHECK("k_aura_fill");
    if (nch_max > 0) {
        static bool attr_dev[kMaxDevices] = {};
        const int smem = (int)(sizeof(LzWarp) * kLzWarps);
        if (!attr_dev[c->device]) {
            BDM_CUDA_TRY(cudaFuncSetAttribute(k_lz4_compress,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr_dev[c->device] = true;
        }
        k_lz4_compress<<<nblk(nch_max, kLzWarps), 32 * kLzWarps, smem, st>>>(
            W.pay, newrank, n, nref, nch_max, W.tmp, W.sizes);
        BDM_LAUNCH_CHECK("k_lz4_compress");
        c->launches += 1;
    }
    if ((s = launch_scan_u32(c, W.sizes, nch_max + 1, st)) != BDM_OK) return s;
    const int64_t thr = 32 * (nch_max > 0 ? nch_max : 1);
    k_aura_pack<<<nblk(thr, 256), 256, 0, st>>>(W.tmp, W.sizes, newrank, n, nref, nch_max, out_cap,
                                                out, W.res);
    BDM_LAUNCH_CHECK("k_aura_pack");
    c->launches += 1;
    long long res[2] = {0, 0};
    BDM_CUDA_TRY(cudaMemcpyAsync(res, W.res, sizeof(res), cudaMemcpyDeviceToHost, st));
    BDM_CUDA_TRY(cudaStreamSynchronize(st));
    *out_size = res[0];
    if (!res[1]) {
        set_error("aura stream needs " + std::to_string(res[0]) + " bytes");
        return BDM_ECAPACITY;
    }
    return BDM_OK;
}

bdm_status launch_aura_decode(Ctx *c, const uint8_t *in, int64_t in_size, const bdm_agents *r,
                              bdm_agents *m, cudaStream_t st) {
    if (in_size < kHdr) {
        set_error("aura stream shorter than its header");
        return BDM_EINVAL;
    }
    AuraHeader h;
    BDM_CUDA_TRY(cudaMemcpyAsync(&h, in, sizeof(h), cudaMemcpyDeviceToHost, st));
    BDM_CUDA_TRY(cudaStreamSynchronize(st));
    const int64_t nref = (int64_t)h.nref, nnew = (int64_t)h.nnew, size = (int64_t)h.size,
                  nch = h.nch;
    if (h.magic != kMagic || h.chunk != (uint32_t)kChunk || nref != r->n ||
        size != payload_size(nref, nnew) || nch != (size + kChunk - 1) / kChunk ||
        in_size < kHdr + 4 * nch) {
        set_error("malformed aura stream (or another reference)");
        return BDM_EINVAL;
    }
    std::vector<uint32_t> len((size_t)nch), off((size_t)nch);
    if (nch > 0)
        BDM_CUDA_TRY(cudaMemcpyAsync(len.data(), in + kHdr, 4 * (size_t)nch,
                                     cudaMemcpyDeviceToHost, st));
    BDM_CUDA_TRY(cudaStreamSynchronize(st));
    int64_t o = kHdr + 4 * nch;
    for (int64_t k = 0; k < nch; ++k) {
        off[(size_t)k] = (uint32_t)o;
        o += len[(size_t)k];
    }
    if (o > in_size) {
        set_error("aura stream truncated");
        return BDM_EINVAL;
    }
    AuraWs &W = c->aura;
    const int64_t nw = (nref + 31) / 32;
    bdm_status s;
    if ((s = ensure(&W.pay, W.pay_cap, size)) != BDM_OK) return s;
    if ((s = ensure(&W.sizes, W.sizes_cap, 2 * nch + 2)) != BDM_OK) return s;
    if ((s = ensure(&W.u32a, W.u32a_cap, nw + 1)) != BDM_OK) return s;
    if ((s = ensure_scan(c, nw + 1)) != BDM_OK) return s;
    if (!W.err) BDM_CUDA_TRY(cudaMalloc(&W.err, sizeof(int)));
    BDM_CUDA_TRY(cudaMemsetAsync(W.err, 0, sizeof(int), st));
    if (nch > 0) {
        BDM_CUDA_TRY(cudaMemcpyAsync(W.sizes, off.data(), 4 * (size_t)nch, cudaMemcpyHostToDevice, st));
        BDM_CUDA_TRY(cudaMemcpyAsync(W.sizes + nch, len.data(), 4 * (size_t)nch,
                                     cudaMemcpyHostToDevice, st));
        k_lz4_decompress<<<nblk(nch, kLzWarps), 32 * kLzWarps, 0, st>>>(
            in, W.sizes, W.sizes + nch, size, nch, W.pay, W.err);
        BDM_LAUNCH_CHECK("k_lz4_decompress");
        c->launches += 1;
    }
    k_aura_presence_counts<<<nblk(nw + 1, 256), 256, 0, st>>>(W.pay, nw, W.u32a);
    c->launches += 1;
    if ((s = launch_scan_u32(c, W.u32a, nw + 1, st)) != BDM_OK) return s;
    int err = 0;
    uint32_t npres = 0;
    BDM_CUDA_TRY(cudaMemcpyAsync(&err, W.err, sizeof(int), cudaMemcpyDeviceToHost, st));
    BDM_CUDA_TRY(cudaMemcpyAsync(&npres, W.u32a + nw, 4, cudaMemcpyDeviceToHost, st));
    BDM_CUDA_TRY(cudaStreamSynchronize(st));
    if (err) {
        set_error("malformed LZ4 block in the aura stream");
        return BDM_EINVAL;
    }
    const int64_t nout = (int64_t)npres + nnew;
    if (nout > m->capacity) {
        set_error("decoded aura needs " + std::to_string((long long)nout) + " agents");
        return BDM_ECAPACITY;
    }
    if (nref + nnew > 0) {
        k_aura_unfill<<<nblk(nref + nnew, 256), 256, 0, st>>>(W.pay, nref, nnew, W.u32a, view(r),
                                                              outv(m));
        BDM_LAUNCH_CHECK("k_aura_unfill");
        c->launches += 1;
    }
    m->n = nout;
    BDM_CUDA_TRY(cudaStreamSynchronize(st));
    return BDM_OK;
}

void free_aura(Ctx *c) {
    AuraWs &W = c->aura;
    void *p[] = {W.u32a, W.u32b, W.pay, W.tmp, W.sizes, W.err, W.res};
    for (void *q : p)
        if (q) cudaFree(q);
    W = AuraWs();
}

}  // namespace bdm
