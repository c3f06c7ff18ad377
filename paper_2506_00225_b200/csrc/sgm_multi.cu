// Multi-GPU pieces of the C ABI: the device snapshot interchange behind the
// map broadcast (collective C1) and a multi-device scorer for single-process callers such
// as the C++ drop-in's refresh_candidate_scores (explorer.cpp:186-205; the reference's
// candidate loop "parallelizes over candidates").
//
// Snapshot blob (device memory, 16-byte aligned segments):
//   header (kHeader bytes: magic, version, n, k, kpad, C, num_classes, dup_idx, aniso)
//   geo [5][ns] f64 | color [ns][4] f64 | idx [ns][kpad] u16 | prob [ns][kpad] f64 |
//   perm [ns][kpad] u16 | (aniso) cov [6][ns] f64
// It is the already-activated, class-sorted device layout, so an imported map is bit-identical
// to the exported one and no rank repeats the host activations (exp / sigmoid with the
// reference's libm) or the row sort.
//
// sgm_multi: one sgm_ctx per device; the map is uploaded once (device 0) and replicated by
// device-to-device copies of the blob (NVLink peer copies where peer access is available);
// views are sharded contiguously (sizes differ by <= 1) and scored by one host thread per
// device; each view's result is written to its own slot of the caller's arrays, so per-view
// results are bit-identical to a single-device call.
#include "sgm_ctx.h"

namespace {

constexpr uint64_t kMagic = 0x53474d42534e4150ull;  // "SGMBSNAP"
constexpr uint64_t kVersion = 1;
constexpr size_t kHeader = 128;

inline size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

struct BlobHeader {
    uint64_t magic, version, n;
    int32_t k, kpad, C, num_classes, dup_idx, aniso;
    uint64_t total;
};
static_assert(sizeof(BlobHeader) <= kHeader, "blob header");

struct Segs {
    size_t geo, color, idx, prob, perm, cov, total;
};

Segs segs_of(uint64_t n, int kpad, bool aniso) {
    const size_t ns = std::max<uint64_t>(n, 1);
    Segs s;
    s.geo = kHeader;
    s.color = s.geo + al16(8 * 5 * ns);
    s.idx = s.color + al16(8 * 4 * ns);
    s.prob = s.idx + al16(2 * ns * kpad);
    s.perm = s.prob + al16(8 * ns * kpad);
    s.cov = s.perm + al16(2 * ns * kpad);
    s.total = s.cov + (aniso ? al16(8 * 6 * ns) : 0);
    return s;
}

}  // namespace

struct sgm_multi {
    std::vector<sgm_ctx*> ctx;
    std::string err;
};

struct sgm_multi_map {
    std::vector<sgm_map*> maps;  // one per device of the sgm_multi, same order
};

extern "C" {

int sgm_map_info(sgm_ctx* ctx, const sgm_map* map, uint64_t* n, int32_t* k, int32_t* num_classes,
                 int32_t* anisotropic) {
    return guard(ctx, [&] {
        if (!map) fail(SGM_ERR_INVALID, "map is null");
        if (n) *n = map->dev.n;
        if (k) *k = map->dev.k;
        if (num_classes) *num_classes = map->num_classes;
        if (anisotropic) *anisotropic = map->dev.aniso;
    });
}

int sgm_map_export_bytes(sgm_ctx* ctx, const sgm_map* map, uint64_t* bytes) {
    return guard(ctx, [&] {
        if (!map || !bytes) fail(SGM_ERR_INVALID, "map / bytes is null");
        *bytes = segs_of(map->dev.n, map->dev.kpad, map->dev.aniso != 0).total;
    });
}

int sgm_map_export(sgm_ctx* ctx, const sgm_map* map, void* d_blob, uint64_t capacity) {
    return guard(ctx, [&] {
        need_ctx(ctx);
        if (!map || !d_blob) fail(SGM_ERR_INVALID, "map / blob is null");
        map_ready(ctx, map);
        const DevMap& d = map->dev;
        const Segs sg = segs_of(d.n, d.kpad, d.aniso != 0);
        if (capacity < sg.total)
            fail(SGM_ERR_INVALID, "blob capacity %llu < %llu bytes",
                 static_cast<unsigned long long>(capacity), static_cast<unsigned long long>(sg.total));
        BlobHeader h{kMagic, kVersion, d.n, d.k, d.kpad, d.C, map->num_classes, d.dup_idx, d.aniso,
                     sg.total};
        char* b = static_cast<char*>(d_blob);
        cudaStream_t s = ctx->stream;
        const size_t ns = std::max<uint64_t>(d.n, 1);
        CK(cudaMemcpyAsync(b, &h, sizeof(h), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(b + sg.geo, map->geo.p, 8 * 5 * ns, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(b + sg.color, map->color.p, 8 * 4 * ns, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(b + sg.idx, map->idx.p, 2 * ns * d.kpad, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(b + sg.prob, map->prob.p, 8 * ns * d.kpad, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(b + sg.perm, map->perm.p, 2 * ns * d.kpad, cudaMemcpyDeviceToDevice, s));
        if (d.aniso) CK(cudaMemcpyAsync(b + sg.cov, map->cov.p, 8 * 6 * ns, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));  // the header lives on this call's stack
    });
}

int sgm_map_import(sgm_ctx* ctx, const void* d_blob, uint64_t bytes, sgm_map** out) {
    sgm_map* m = nullptr;
    int rc = guard(ctx, [&] {
        need_ctx(ctx);
        if (!d_blob || !out) fail(SGM_ERR_INVALID, "blob / out is null");
        *out = nullptr;
        if (bytes < kHeader) fail(SGM_ERR_INVALID, "blob of %llu bytes has no header",
                                  static_cast<unsigned long long>(bytes));
        const char* b = static_cast<const char*>(d_blob);
        BlobHeader h{};
        CK(cudaMemcpy(&h, b, sizeof(h), cudaMemcpyDefault));
        if (h.magic != kMagic || h.version != kVersion) fail(SGM_ERR_INVALID, "not a map snapshot blob");
        const Segs sg = segs_of(h.n, h.kpad, h.aniso != 0);
        if (h.total != sg.total || bytes < sg.total)
            fail(SGM_ERR_INVALID, "snapshot blob truncated (%llu of %llu bytes)",
                 static_cast<unsigned long long>(bytes), static_cast<unsigned long long>(sg.total));
        m = new sgm_map();
        m->num_classes = h.num_classes;
        const size_t ns = std::max<uint64_t>(h.n, 1);
        cudaStream_t s = ctx->stream;
        ctx->take(m->geo, 8 * 5 * ns);
        ctx->take(m->color, 8 * 4 * ns);
        ctx->take(m->idx, 2 * ns * h.kpad);
        ctx->take(m->prob, 8 * ns * h.kpad);
        ctx->take(m->perm, 2 * ns * h.kpad);
        CK(m->geo.reserve(8 * 5 * ns));
        CK(m->color.reserve(8 * 4 * ns));
        CK(m->idx.reserve(2 * ns * h.kpad));
        CK(m->prob.reserve(8 * ns * h.kpad));
        CK(m->perm.reserve(2 * ns * h.kpad));
        // cudaMemcpyDefault: the blob may sit on another device (peer copy over NVLink)
        CK(cudaMemcpyAsync(m->geo.p, b + sg.geo, 8 * 5 * ns, cudaMemcpyDefault, s));
        CK(cudaMemcpyAsync(m->color.p, b + sg.color, 8 * 4 * ns, cudaMemcpyDefault, s));
        CK(cudaMemcpyAsync(m->idx.p, b + sg.idx, 2 * ns * h.kpad, cudaMemcpyDefault, s));
        CK(cudaMemcpyAsync(m->prob.p, b + sg.prob, 8 * ns * h.kpad, cudaMemcpyDefault, s));
        CK(cudaMemcpyAsync(m->perm.p, b + sg.perm, 2 * ns * h.kpad, cudaMemcpyDefault, s));
        if (h.aniso) {
            ctx->take(m->cov, 8 * 6 * ns);
            CK(m->cov.reserve(8 * 6 * ns));
            CK(cudaMemcpyAsync(m->cov.p, b + sg.cov, 8 * 6 * ns, cudaMemcpyDefault, s));
        }
        CK(cudaStreamSynchronize(s));
        DevMap& d = m->dev;
        d.n = h.n;
        d.k = h.k;
        d.kpad = h.kpad;
        d.C = h.C;
        const double* g = m->geo.as<double>();
        d.cx = g;
        d.cy = g + ns;
        d.cz = g + 2 * ns;
        d.rad = g + 3 * ns;
        d.alpha = g + 4 * ns;
        d.color4 = m->color.as<double>();
        d.sem_idx = m->idx.as<uint16_t>();
        d.sem_prob = m->prob.as<double>();
        d.sem_perm = m->perm.as<uint16_t>();
        d.dup_idx = h.dup_idx;
        d.aniso = h.aniso;
        d.cov = h.aniso ? m->cov.as<double>() : nullptr;
        m->groups = choose_groups(h.C, h.k);
        map_group_bounds(ctx, m, s);
        *out = m;
        m = nullptr;
    });
    delete m;
    return rc;
}

// ---- sgm_multi ----

static int multi_guard(sgm_multi* mg, const std::function<void()>& fn) {
    try {
        fn();
        if (mg) mg->err.clear();
        return SGM_OK;
    } catch (const SgmError& e) {
        if (mg) mg->err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        if (mg) mg->err = "host allocation failed";
        return SGM_ERR_OOM;
    } catch (const std::exception& e) {
        if (mg) mg->err = e.what();
        return SGM_ERR_INVALID;
    }
}

int sgm_multi_create(int32_t n_devices, const int32_t* devices, sgm_multi** out) {
    if (!out) return SGM_ERR_INVALID;
    *out = nullptr;
    auto* mg = new (std::nothrow) sgm_multi();
    if (!mg) return SGM_ERR_OOM;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    if (n_devices <= 0) n_devices = count;  // all visible devices
    if (n_devices <= 0) {
        sgm_ctx* probe = nullptr;  // reports "no CUDA device" through sgm_last_error(NULL)
        const int rc = sgm_ctx_create(0, &probe);
        delete mg;
        return rc != SGM_OK ? rc : SGM_ERR_CUDA;
    }
    for (int i = 0; i < n_devices; ++i) {
        sgm_ctx* c = nullptr;
        const int rc = sgm_ctx_create(devices ? devices[i] : i, &c);
        if (rc != SGM_OK) {  // sgm_last_error(NULL) holds the reason
            for (sgm_ctx* x : mg->ctx) sgm_ctx_destroy(x);
            delete mg;
            return rc;
        }
        mg->ctx.push_back(c);
    }
    // NVLink peer access between the devices (the replication and a peer-resident blob)
    for (size_t i = 0; i < mg->ctx.size(); ++i)
        for (size_t j = 0; j < mg->ctx.size(); ++j) {
            const int a = mg->ctx[i]->device, b = mg->ctx[j]->device;
            int can = 0;
            if (a != b && cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
                cudaSetDevice(a);
                if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already on
            }
        }
    *out = mg;
    return SGM_OK;
}

void sgm_multi_destroy(sgm_multi* mg) {
    if (!mg) return;
    for (sgm_ctx* c : mg->ctx) sgm_ctx_destroy(c);
    delete mg;
}

const char* sgm_multi_last_error(const sgm_multi* mg) { return mg ? mg->err.c_str() : ""; }

int32_t sgm_multi_device_count(const sgm_multi* mg) {
    return mg ? static_cast<int32_t>(mg->ctx.size()) : 0;
}

sgm_ctx* sgm_multi_ctx(sgm_multi* mg, int32_t i) {
    if (!mg || i < 0 || i >= static_cast<int32_t>(mg->ctx.size())) return nullptr;
    return mg->ctx[i];
}

void sgm_multi_map_release(sgm_multi* mg, sgm_multi_map* mm) {
    if (!mm) return;
    for (size_t i = 0; i < mm->maps.size(); ++i)
        sgm_map_release(mg && i < mg->ctx.size() ? mg->ctx[i] : nullptr, mm->maps[i]);
    delete mm;
}

int sgm_multi_map_upload(sgm_multi* mg, uint64_t n, int32_t k, int32_t num_classes,
                         const double* centers, const double* log_radii,
                         const double* opacity_logits, const double* colors,
                         const uint16_t* sem_indices, const double* sem_probs,
                         sgm_multi_map** out) {
    sgm_multi_map* mm = nullptr;
    int rc = multi_guard(mg, [&] {
        if (!mg || !out) fail(SGM_ERR_INVALID, "multi / out is null");
        *out = nullptr;
        mm = new sgm_multi_map();
        mm->maps.assign(mg->ctx.size(), nullptr);
        sgm_ctx* c0 = mg->ctx[0];
        auto chk = [&](sgm_ctx* c, int code) {
            if (code != SGM_OK) throw SgmError{code, c->err};
        };
        // one upload (host activations + H2D + row sort) on the first device ...
        chk(c0, sgm_map_upload(c0, n, k, num_classes, centers, log_radii, opacity_logits, colors,
                               sem_indices, sem_probs, &mm->maps[0]));
        if (mg->ctx.size() == 1) return;
        // ... then the device snapshot is replicated device to device (C1)
        uint64_t bytes = 0;
        chk(c0, sgm_map_export_bytes(c0, mm->maps[0], &bytes));
        CK(cudaSetDevice(c0->device));
        DevBuf blob;
        CK(blob.reserve(bytes));
        chk(c0, sgm_map_export(c0, mm->maps[0], blob.p, bytes));
        for (size_t i = 1; i < mg->ctx.size(); ++i)
            chk(mg->ctx[i], sgm_map_import(mg->ctx[i], blob.p, bytes, &mm->maps[i]));
        CK(cudaSetDevice(c0->device));  // blob freed on its own device
    });
    if (rc == SGM_OK) {
        *out = mm;
    } else {
        sgm_multi_map_release(mg, mm);
    }
    return rc;
}

// Shards n views over the devices and scores them concurrently (one host thread per device).
static int multi_score(sgm_multi* mg, const sgm_multi_map* mm, const sgm_camera* cam, uint64_t n,
                       const sgm_pose* poses, const sgm_candidate* cands, const sgm_options* opt,
                       double* n_missing, double* entropy_sum) {
    return multi_guard(mg, [&] {
        if (!mg || !mm || mm->maps.size() != mg->ctx.size()) fail(SGM_ERR_INVALID, "multi / map mismatch");
        if (n > 0 && (!n_missing || !entropy_sum || (!poses && !cands)))
            fail(SGM_ERR_INVALID, "null view or output array");
        const size_t D = mg->ctx.size();
        std::vector<int> rcs(D, SGM_OK);
        auto work = [&](size_t r) {
            const uint64_t base = n / D, rem = n % D;
            const uint64_t s = r * base + std::min<uint64_t>(r, rem);
            const uint64_t e = s + base + (r < rem ? 1 : 0);
            if (e == s) return;
            sgm_ctx* c = mg->ctx[r];
            rcs[r] = poses ? sgm_score_views(c, mm->maps[r], cam, e - s, poses + s, opt,
                                             n_missing + s, entropy_sum + s)
                           : sgm_score_candidates(c, mm->maps[r], cam, e - s, cands + s, opt,
                                                  n_missing + s, entropy_sum + s);
        };
        std::vector<std::thread> th;
        for (size_t r = 1; r < D; ++r) th.emplace_back(work, r);
        work(0);
        for (auto& t : th) t.join();
        for (size_t r = 0; r < D; ++r)
            if (rcs[r] != SGM_OK)
                fail(rcs[r], "device %d: %s", mg->ctx[r]->device, mg->ctx[r]->err.c_str());
    });
}

int sgm_multi_score_views(sgm_multi* mg, const sgm_multi_map* map, const sgm_camera* cam,
                          uint64_t n, const sgm_pose* poses, const sgm_options* opt,
                          double* n_missing, double* entropy_sum) {
    return multi_score(mg, map, cam, n, poses, nullptr, opt, n_missing, entropy_sum);
}

int sgm_multi_score_candidates(sgm_multi* mg, const sgm_multi_map* map, const sgm_camera* cam,
                               uint64_t n, const sgm_candidate* cands, const sgm_options* opt,
                               double* n_missing, double* entropy_sum) {
    return multi_score(mg, map, cam, n, nullptr, cands, opt, n_missing, entropy_sum);
}

}  // extern "C"
