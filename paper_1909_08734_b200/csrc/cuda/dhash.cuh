// Device open-addressing hash tables for the device setup (setup_dev.cu):
// 64-bit keys (0 = empty slot), int32 values, linear probing, insertion by
// atomicCAS.  Used for lattice sets (band, BFS "seen", ghosts), the band's
// lattice -> code map, (subdomain, node) membership sets and mesh cells.
#pragma once

#include "common.cuh"

#include <cstdint>

namespace cpddg {

__host__ __device__ __forceinline__ std::uint64_t dhash_mix(std::uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ULL;
    k ^= k >> 33;
    return k;
}

/** View of a device table (passed to kernels by value). */
struct DHash {
    unsigned long long* keys = nullptr;
    int* vals = nullptr;
    unsigned long long mask = 0;

    __device__ __forceinline__ int find(std::uint64_t key) const {
        unsigned long long i = dhash_mix(key) & mask;
        for (;;) {
            const unsigned long long k = keys[i];
            if (k == key) return vals[i];
            if (k == 0) return -1;
            i = (i + 1) & mask;
        }
    }
    __device__ __forceinline__ bool contains(std::uint64_t key) const {
        unsigned long long i = dhash_mix(key) & mask;
        for (;;) {
            const unsigned long long k = keys[i];
            if (k == key) return true;
            if (k == 0) return false;
            i = (i + 1) & mask;
        }
    }
    /** Insert key; true if this call inserted it (then vals[slot] = val). */
    __device__ __forceinline__ bool insert(std::uint64_t key, int val) {
        unsigned long long i = dhash_mix(key) & mask;
        for (;;) {
            const unsigned long long prev = atomicCAS(keys + i, 0ULL, static_cast<unsigned long long>(key));
            if (prev == 0) {
                vals[i] = val;
                return true;
            }
            if (prev == key) return false;
            i = (i + 1) & mask;
        }
    }
    /** Insert key; if this call inserted it, claim the next position of
     *  *counter as its value and return it, else return -1. */
    __device__ __forceinline__ int insert_claim(std::uint64_t key, int* counter) {
        unsigned long long i = dhash_mix(key) & mask;
        for (;;) {
            const unsigned long long prev = atomicCAS(keys + i, 0ULL, static_cast<unsigned long long>(key));
            if (prev == 0) {
                const int pos = atomicAdd(counter, 1);
                vals[i] = pos;
                return pos;
            }
            if (prev == key) return -1;
            i = (i + 1) & mask;
        }
    }
};

/** Owning device table with capacity a power of two >= 2 x the expected size. */
struct DevHashTable {
    DevBuf<unsigned long long> keys;
    DevBuf<int> vals;
    unsigned long long cap = 0;
    void init(std::size_t expected, cudaStream_t st = nullptr) {
        unsigned long long c = 1024;
        while (c < 2 * static_cast<unsigned long long>(expected)) c <<= 1;
        if (c != cap) {
            keys.alloc(c);
            vals.alloc(c);
            cap = c;
        }
        keys.zero(st);
    }
    DHash view() const {
        DHash h;
        h.keys = keys.get();
        h.vals = vals.get();
        h.mask = cap - 1;
        return h;
    }
};

}  // namespace cpddg
