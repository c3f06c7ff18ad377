// Exploration map on the GPU: ExplorationMap::integrate_frame,
// seed_*_region and the lattice test of sample_candidates
// (proj/src/explorer.cpp:11-184), bit-identical to the reference.
//
// The reference walks rays one after another and mutates the grid in place:
//   mark_free:     unknown -> free (+ changelog append)      explorer.cpp:38-43
//   mark_occupied: any     -> occupied                        explorer.cpp:45-51
// Both transitions are monotone, so the final state of a voxel does not depend on
// the ray order: occupied if any ray hit it, else free if any ray crossed it. Only
// the changelog depends on order: a voxel unknown before the frame is logged iff
// its first event in sequential order is a crossing, and the log is ordered by
// that first crossing. Sequential order is (ray r, step s) with the hit of ray r
// after all of its steps (:95-107), so:
//   pass 1 (one thread per ray): the exact fp64 walk of :56-106; a crossing of a
//          pre-frame-unknown voxel does atomicMin(first_free[v], r<<32 | s), a hit
//          of a non-occupied voxel does atomicMin(first_hit[v], r)
//   pass 2 (one thread per voxel): new state, logged iff first_free.r < first_hit,
//          emitted as (key = first_free, id) and sorted by key on the host side.
// Compiled with --fmad=false: every fp64 expression is evaluated with one rounding
// per operation in the reference's order (Eigen 3-term products as x0 + (x1 + x2)).
#include <climits>

#include "sgm_internal.h"

namespace sgm {

namespace {

constexpr uint8_t kUnknown = 0, kFree = 1, kOccupied = 2;  // VoxelState, explorer.hpp:11

__device__ __forceinline__ int to_int_x86(double v) {
    return (v > -2147483649.0 && v < 2147483648.0) ? static_cast<int>(v) : INT_MIN;
}

__device__ __forceinline__ bool in_grid(const EmapParams& e, int ix, int iy, int iz) {
    return ix >= 0 && iy >= 0 && iz >= 0 && ix < e.dims[0] && iy < e.dims[1] && iz < e.dims[2];
}

__device__ __forceinline__ int linear_index(const EmapParams& e, int ix, int iy, int iz) {
    return (iz * e.dims[1] + iy) * e.dims[0] + ix;  // explorer.hpp:25-27
}

// ExplorationMap::voxel_at, explorer.cpp:22-29.
__device__ __forceinline__ int voxel_at(const EmapParams& e, double px, double py, double pz) {
    const int ix = to_int_x86(floor((px - e.origin[0]) / e.voxel));
    const int iy = to_int_x86(floor((py - e.origin[1]) / e.voxel));
    const int iz = to_int_x86(floor((pz - e.origin[2]) / e.voxel));
    if (!in_grid(e, ix, iy, iz)) return -1;
    return linear_index(e, ix, iy, iz);
}

// Pass 1: one thread per strided depth pixel, explorer.cpp:55-107.
__global__ void __launch_bounds__(256) k_emap_rays(EmapParams e, CamParams cam, WorldPose P,
                                                   const float* __restrict__ depth, int stride,
                                                   int nx, int nrays,
                                                   const uint8_t* __restrict__ grid,
                                                   unsigned long long* __restrict__ first_free,
                                                   uint32_t* __restrict__ first_hit) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrays) return;
    const int x = (r % nx) * stride, y = (r / nx) * stride;
    const float d = depth[static_cast<size_t>(y) * cam.W + x];
    if (d <= 0) return;  // :58 (NaN passes, as in the reference)
    const double dd = static_cast<double>(d);
    // end = pose.to_world(camera.pixel_ray(x, y) * d)   camera.hpp:45-47, geometry.hpp:22
    const double c0 = (x + 0.5 - cam.cx) / cam.fx * dd;
    const double c1 = (y + 0.5 - cam.cy) / cam.fy * dd;
    const double c2 = 1.0 * dd;
    double end[3], dir[3];
    const double start[3] = {P.t[0], P.t[1], P.t[2]};
#pragma unroll
    for (int i = 0; i < 3; ++i)
        end[i] = (P.R[3 * i] * c0 + (P.R[3 * i + 1] * c1 + P.R[3 * i + 2] * c2)) + P.t[i];
    int idx[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) idx[a] = to_int_x86(floor((start[a] - e.origin[a]) / e.voxel));
#pragma unroll
    for (int a = 0; a < 3; ++a) dir[a] = end[a] - start[a];
    const double len = sqrt(dir[0] * dir[0] + (dir[1] * dir[1] + dir[2] * dir[2]));
    if (len < 1e-12) return;  // :68
#pragma unroll
    for (int a = 0; a < 3; ++a) dir[a] = dir[a] / len;
    // :72 hit classified by a point just inside the surface
    const int hit = voxel_at(e, end[0] - dir[0] * 1e-6, end[1] - dir[1] * 1e-6,
                             end[2] - dir[2] * 1e-6);
    int step[3];
    double t_max[3], t_delta[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {  // :77-89
        if (fabs(dir[a]) < 1e-12) {
            step[a] = 0;
            t_max[a] = 1e300;
            t_delta[a] = 1e300;
        } else {
            step[a] = dir[a] > 0 ? 1 : -1;
            const double boundary = e.origin[a] + (idx[a] + (dir[a] > 0 ? 1.0 : 0.0)) * e.voxel;
            t_max[a] = (boundary - start[a]) / dir[a];
            t_delta[a] = e.voxel / fabs(dir[a]);
        }
    }
    double t = 0.0;
    int guard = e.dims[0] + e.dims[1] + e.dims[2] + 4;
    const unsigned long long rk = static_cast<unsigned long long>(r) << 32;
    uint32_t s = 0;
    while (guard-- > 0 && t <= len) {  // :93-104
        if (!in_grid(e, idx[0], idx[1], idx[2])) break;
        const int id = linear_index(e, idx[0], idx[1], idx[2]);
        if (id == hit) break;
        if (grid[id] == kUnknown) atomicMin(&first_free[id], rk | s);  // mark_free
        ++s;
        int axis = 0;
        if (t_max[1] < t_max[axis]) axis = 1;
        if (t_max[2] < t_max[axis]) axis = 2;
        t = t_max[axis];
        t_max[axis] += t_delta[axis];
        idx[axis] += step[axis];
    }
    if (hit >= 0 && grid[hit] != kOccupied) atomicMin(&first_hit[hit], static_cast<uint32_t>(r));
}

// Seeding, explorer.cpp:124-132: ids ascending, so the changelog key is the id.
__global__ void k_emap_seed(EmapParams e, sgm_aabb box, int occupied, const uint8_t* grid,
                            unsigned long long* first_free, uint32_t* first_hit) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= e.nvox) return;
    const int id = static_cast<int>(i);
    const int ix = id % e.dims[0];  // voxel_center, :31-36
    const int iy = (id / e.dims[0]) % e.dims[1];
    const int iz = id / (e.dims[0] * e.dims[1]);
    const double p[3] = {e.origin[0] + e.voxel * (ix + 0.5), e.origin[1] + e.voxel * (iy + 0.5),
                         e.origin[2] + e.voxel * (iz + 0.5)};
    bool in = true;  // Aabb::contains, geometry.hpp:64-66
#pragma unroll
    for (int a = 0; a < 3; ++a) in = in && p[a] >= box.min[a] && p[a] <= box.max[a];
    if (!in) return;
    if (occupied) {
        if (grid[i] != kOccupied) first_hit[i] = 0;
    } else if (grid[i] == kUnknown) {
        first_free[i] = static_cast<unsigned long long>(i);
    }
}

// Pass 2: apply, count, emit new changelog entries; resets the scratch it read.
__global__ void __launch_bounds__(256) k_emap_resolve(uint64_t nvox, uint8_t* __restrict__ grid,
                                                      unsigned long long* __restrict__ first_free,
                                                      uint32_t* __restrict__ first_hit,
                                                      unsigned long long* __restrict__ log_keys,
                                                      int32_t* __restrict__ log_ids,
                                                      unsigned long long* __restrict__ counters) {
    // counters: [0] new log entries, [1] free voxels, [2] occupied voxels
    unsigned nfree = 0, nocc = 0;
    const int lane = threadIdx.x & 31;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
         i - lane < nvox; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        bool emit = false;
        unsigned long long key = 0;
        if (i < nvox) {
            const uint8_t s0 = grid[i];
            const unsigned long long f = first_free[i];
            const uint32_t h = first_hit[i];
            uint8_t s1 = s0;
            if (h != 0xffffffffu) s1 = kOccupied;
            else if (f != ~0ull) s1 = kFree;
            if (s1 != s0) grid[i] = s1;
            if (f != ~0ull) first_free[i] = ~0ull;
            if (h != 0xffffffffu) first_hit[i] = 0xffffffffu;
            emit = s0 == kUnknown && f != ~0ull && (f >> 32) < h;
            key = f;
            nfree += s1 == kFree;
            nocc += s1 == kOccupied;
        }
        const unsigned mask = __ballot_sync(0xffffffffu, emit);
        if (mask) {
            unsigned long long base = 0;
            if (lane == __ffs(mask) - 1) base = atomicAdd(&counters[0], __popc(mask));
            base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
            if (emit) {
                const unsigned long long pos = base + __popc(mask & ((1u << lane) - 1));
                log_keys[pos] = key;
                log_ids[pos] = static_cast<int32_t>(i);
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        nfree += __shfl_xor_sync(0xffffffffu, nfree, o);
        nocc += __shfl_xor_sync(0xffffffffu, nocc, o);
    }
    if (lane == 0) {
        if (nfree) atomicAdd(&counters[1], static_cast<unsigned long long>(nfree));
        if (nocc) atomicAdd(&counters[2], static_cast<unsigned long long>(nocc));
    }
}

// Lattice test of sample_candidates (explorer.cpp:171-174) plus the fresh set.
__global__ void k_emap_lattice(EmapParams e, const double* __restrict__ pos, int n,
                               const uint8_t* __restrict__ grid, const uint8_t* __restrict__ fresh,
                               uint8_t* __restrict__ ok) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int id = voxel_at(e, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2]);
    ok[j] = id >= 0 && grid[id] == kFree && fresh[id];
}

__global__ void k_emap_mark(const int32_t* __restrict__ ids, uint64_t n, uint8_t* flags,
                            uint8_t value) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n) flags[ids[i]] = value;
}

__global__ void k_emap_free_ids(uint64_t nvox, const uint8_t* __restrict__ grid,
                                unsigned long long* __restrict__ log_keys,
                                int32_t* __restrict__ log_ids, unsigned long long* counter) {
    const int lane = threadIdx.x & 31;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
         i - lane < nvox; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const bool emit = i < nvox && grid[i] == kFree;
        const unsigned mask = __ballot_sync(0xffffffffu, emit);
        if (!mask) continue;
        unsigned long long base = 0;
        if (lane == __ffs(mask) - 1) base = atomicAdd(counter, __popc(mask));
        base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
        if (emit) {
            const unsigned long long pos = base + __popc(mask & ((1u << lane) - 1));
            log_keys[pos] = i;
            log_ids[pos] = static_cast<int32_t>(i);
        }
    }
}

int grid_blocks(uint64_t n) {
    const uint64_t b = (n + 255) / 256;
    return static_cast<int>(b < 148ull * 16 ? (b ? b : 1) : 148ull * 16);
}

}  // namespace

void launch_emap_rays(const EmapParams& e, const CamParams& cam, const WorldPose& P,
                      const float* depth, int stride, const uint8_t* grid,
                      unsigned long long* first_free, uint32_t* first_hit, cudaStream_t s) {
    const int nx = (cam.W + stride - 1) / stride, ny = (cam.H + stride - 1) / stride;
    const int nrays = nx * ny;
    if (nrays == 0) return;
    k_emap_rays<<<(nrays + 255) / 256, 256, 0, s>>>(e, cam, P, depth, stride, nx, nrays, grid,
                                                    first_free, first_hit);
}

void launch_emap_seed(const EmapParams& e, const sgm_aabb& box, int occupied, const uint8_t* grid,
                      unsigned long long* first_free, uint32_t* first_hit, cudaStream_t s) {
    k_emap_seed<<<static_cast<unsigned>((e.nvox + 255) / 256), 256, 0, s>>>(
        e, box, occupied, grid, first_free, first_hit);
}

void launch_emap_resolve(const EmapParams& e, uint8_t* grid, unsigned long long* first_free,
                         uint32_t* first_hit, unsigned long long* log_keys, int32_t* log_ids,
                         unsigned long long* counters, cudaStream_t s) {
    k_emap_resolve<<<grid_blocks(e.nvox), 256, 0, s>>>(e.nvox, grid, first_free, first_hit,
                                                       log_keys, log_ids, counters);
}

void launch_emap_lattice(const EmapParams& e, const double* pos, int n, const uint8_t* grid,
                         const uint8_t* fresh, uint8_t* ok, cudaStream_t s) {
    if (n > 0) k_emap_lattice<<<(n + 255) / 256, 256, 0, s>>>(e, pos, n, grid, fresh, ok);
}

void launch_emap_mark(const int32_t* ids, uint64_t n, uint8_t* flags, uint8_t value,
                      cudaStream_t s) {
    if (n > 0)
        k_emap_mark<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(ids, n, flags, value);
}

void launch_emap_free_ids(const EmapParams& e, const uint8_t* grid, unsigned long long* log_keys,
                          int32_t* log_ids, unsigned long long* counter, cudaStream_t s) {
    k_emap_free_ids<<<grid_blocks(e.nvox), 256, 0, s>>>(e.nvox, grid, log_keys, log_ids, counter);
}

}  // namespace sgm
