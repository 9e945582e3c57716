// n-body C ABI (tools/nbody/runner.cpp + steps.hpp on device views).
#include "capi_internal.hpp"

#include <cstring>
#include <memory>
#include <string>
#include <random>
#include <vector>

namespace lamk
{
    cudaError_t nbody_update(const lamp_view* v, bool f64, bool exact, bool phys, uint64_t n, uint64_t ib, uint64_t ie,
                             cudaStream_t s);
    cudaError_t nbody_move(const lamp_view* v, bool f64, bool phys, uint64_t ib, uint64_t ie, cudaStream_t s);
    cudaError_t nbody_account(const lamp_view* v, bool move, uint64_t n, uint64_t ib, uint64_t ie, cudaStream_t s);
    cudaError_t nbody_update_multi(const lamp_view* v, bool f64, bool exact, bool phys, const lamp_view* const* jv,
                                   const uint64_t* jb, const uint64_t* je, size_t nj, uint64_t ib, uint64_t ie,
                                   cudaStream_t s);
    cudaError_t nbody_pack(const lamp_view* v, bool f64, bool phys, uint64_t ib, uint64_t ie, bool withMass, void* out,
                           cudaStream_t s);
    cudaError_t nbody_manual_update(bool soa, bool f64, bool exact, void* base, uint64_t n, cudaStream_t s);
    cudaError_t nbody_manual_move(bool soa, bool f64, void* base, uint64_t n, cudaStream_t s);
} // namespace lamk

// the hand-written baselines' state: one device buffer, AoS records or 7 arrays
struct lam_nbody_manual
{
    bool soa = false, f64 = false;
    uint64_t n = 0;
    int device = 0;
    void* buf = nullptr;
};

using namespace lamb;
using namespace lamhost;

namespace
{
    // the particle record: 7 leaves Pos.{x,y,z}, Vel.{x,y,z}, Mass of one float type
    // (runner.cpp:328-331, accessors.hpp:13-20)
    bool particleF64(const lam_view* v)
    {
        const auto& s = v->L->map->schema();
        if(s.leafCount() != 7)
            throw std::invalid_argument("n-body needs the 7-leaf particle record Pos{x,y,z}, Vel{x,y,z}, Mass");
        const int t = s.leaves()[0].type;
        if(t != F32 && t != F64)
            throw std::invalid_argument("n-body leaves must be f32 or f64");
        for(size_t f = 1; f < 7; ++f)
            if(s.leaves()[f].type != t)
                throw std::invalid_argument("type mismatch: n-body leaves must share one float type");
        return t == F64;
    }

    // every particle leaf an aligned physical leaf: the kernels take the direct-load path
    bool particlePhys(const lam_view* v)
    {
        for(size_t f = 0; f < 7; ++f)
        {
            const lamp_node& nd = v->L->nodes[v->L->roots[f]];
            if(nd.kind != LAMP_PHYS || !(nd.flags & LAMP_FLAG_ALIGNED))
                return false;
        }
        return true;
    }

    struct TempView
    {
        std::shared_ptr<Lowered> L;
        lam_view v;
        void* buf = nullptr;
        TempView(const lam_view& like, int device)
        {
            const Map& m = *like.L->map;
            Factory aos = [](Schema s, Extents e) -> MapPtr { return std::make_shared<AoSMap>(s, e, false); };
            L = lower(aos(m.schema(), m.extents()));
            v.L = L;
            v.device = device;
            v.owned = false;
            const uint64_t bytes = L->map->blobSize(0);
            lam_cuda_check(cudaMalloc(&buf, bytes ? bytes : 16), "cudaMalloc(temp view)");
            v.blobs = {buf};
            v.img.build(*L, device, streamPtrsFor(*L, v.blobs));
        }
        ~TempView()
        {
            v.img.release();
            if(buf)
                cudaFree(buf);
        }
    };

    template<typename F>
    int guard2(F&& f)
    {
        try
        {
            f();
            return LAM_OK;
        }
        catch(const std::invalid_argument& e)
        {
            g_lam_err = e.what();
            return LAM_EINVAL;
        }
        catch(const std::out_of_range& e)
        {
            g_lam_err = e.what();
            return LAM_ERANGE;
        }
        catch(const std::logic_error& e)
        {
            g_lam_err = e.what();
            return LAM_ELOGIC;
        }
        catch(const std::exception& e)
        {
            g_lam_err = e.what();
            return std::string(e.what()).find("cuda") != std::string::npos ? LAM_ECUDA : LAM_ERUNTIME;
        }
    }
} // namespace

extern "C"
{
    int lam_nbody_init(lam_view* v, uint64_t seed, void* stream)
    {
        return guard2(
            [&]
            {
                const bool f64 = particleF64(v);
                DeviceGuard g(v->device);
                const uint64_t n = v->L->map->elementCount();
                auto s = static_cast<cudaStream_t>(stream);
                // drawInitValues (runner.cpp:30-43) then initView (runner.cpp:46-58)
                std::mt19937_64 gen(seed);
                const size_t T = f64 ? 8 : 4;
                std::vector<uint8_t> host(n * 7 * T);
                for(uint64_t i = 0; i < n; ++i)
                {
                    double d[7];
                    d[0] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                    d[1] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                    d[2] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                    d[6] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                    d[3] = d[4] = d[5] = 0.0;
                    for(int f = 0; f < 7; ++f)
                    {
                        if(f64)
                            std::memcpy(&host[(i * 7 + f) * 8], &d[f], 8);
                        else
                        {
                            const float x = static_cast<float>(d[f]);
                            std::memcpy(&host[(i * 7 + f) * 4], &x, 4);
                        }
                    }
                }
                TempView tmp(*v, v->device);
                if(!host.empty())
                    lam_cuda_check(cudaMemcpyAsync(tmp.buf, host.data(), host.size(), cudaMemcpyHostToDevice, s),
                                   "h2d");
                copyViews(tmp.v, *v, 0, n, s);
                lam_cuda_check(cudaStreamSynchronize(s), "sync");
            });
    }

    // ---- hand-written baselines (steps.hpp:124-230, runner.cpp:239-323) -------------------
    int lam_nbody_manual_create(const char* kind, uint64_t n, int f64, uint64_t seed, int device, void* stream,
                                lam_nbody_manual** out)
    {
        return guard2(
            [&]
            {
                const std::string k = kind ? kind : "";
                if(k != "manual-aos" && k != "manual-soa")
                    throw std::invalid_argument("unknown manual baseline: '" + k + "' (manual-aos | manual-soa)");
                auto m = std::make_unique<lam_nbody_manual>();
                m->soa = k == "manual-soa";
                m->f64 = f64 != 0;
                m->n = n;
                m->device = device;
                DeviceGuard g(device);
                const size_t T = m->f64 ? 8 : 4;
                // drawInitValues (runner.cpp:30-43), laid out as ManualParticle[] or ManualSoA
                std::mt19937_64 gen(seed);
                std::vector<uint8_t> host(n * 7 * T);
                for(uint64_t i = 0; i < n; ++i)
                {
                    double d[7];
                    d[0] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                    d[1] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                    d[2] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                    d[6] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                    d[3] = d[4] = d[5] = 0.0;
                    for(int f = 0; f < 7; ++f)
                    {
                        const uint64_t at = m->soa ? (f * n + i) * T : (i * 7 + f) * T;
                        if(m->f64)
                            std::memcpy(&host[at], &d[f], 8);
                        else
                        {
                            const float x = static_cast<float>(d[f]);
                            std::memcpy(&host[at], &x, 4);
                        }
                    }
                }
                lam_cuda_check(cudaMalloc(&m->buf, host.empty() ? 16 : host.size()), "cudaMalloc(manual)");
                auto s = static_cast<cudaStream_t>(stream);
                if(!host.empty())
                    lam_cuda_check(cudaMemcpyAsync(m->buf, host.data(), host.size(), cudaMemcpyHostToDevice, s), "h2d");
                lam_cuda_check(cudaStreamSynchronize(s), "sync");
                *out = m.release();
            });
    }

    int lam_nbody_manual_update(lam_nbody_manual* m, int mode, void* stream)
    {
        return guard2(
            [&]
            {
                DeviceGuard g(m->device);
                lam_cuda_check(lamk::nbody_manual_update(m->soa, m->f64, mode == LAM_NBODY_EXACT, m->buf, m->n,
                                                         static_cast<cudaStream_t>(stream)),
                               "nbody_manual_update");
            });
    }

    int lam_nbody_manual_move(lam_nbody_manual* m, void* stream)
    {
        return guard2(
            [&]
            {
                DeviceGuard g(m->device);
                lam_cuda_check(lamk::nbody_manual_move(m->soa, m->f64, m->buf, m->n, static_cast<cudaStream_t>(stream)),
                               "nbody_manual_move");
            });
    }

    // the checksum of runManual (runner.cpp:303-318): Σ (x, y, z) in double, index order
    int lam_nbody_manual_checksum(const lam_nbody_manual* m, double* out)
    {
        return guard2(
            [&]
            {
                DeviceGuard g(m->device);
                lam_cuda_check(cudaDeviceSynchronize(), "sync");
                const size_t T = m->f64 ? 8 : 4;
                std::vector<uint8_t> host(m->n * 7 * T);
                if(!host.empty())
                    lam_cuda_check(cudaMemcpy(host.data(), m->buf, host.size(), cudaMemcpyDeviceToHost), "d2h");
                double sum = 0;
                for(uint64_t i = 0; i < m->n; ++i)
                    for(int f = 0; f < 3; ++f)
                    {
                        const uint64_t at = m->soa ? (f * m->n + i) * T : (i * 7 + f) * T;
                        if(m->f64)
                        {
                            double x;
                            std::memcpy(&x, &host[at], 8);
                            sum += x;
                        }
                        else
                        {
                            float x;
                            std::memcpy(&x, &host[at], 4);
                            sum += static_cast<double>(x);
                        }
                    }
                *out = sum;
            });
    }

    void lam_nbody_manual_free(lam_nbody_manual* m)
    {
        if(!m)
            return;
        if(m->buf)
        {
            DeviceGuard g(m->device);
            cudaFree(m->buf);
        }
        delete m;
    }

    int lam_nbody_update(lam_view* v, int mode, uint64_t ib, uint64_t ie, void* stream)
    {
        return guard2(
            [&]
            {
                const bool f64 = particleF64(v);
                const uint64_t n = v->L->map->elementCount();
                if(ib > ie || ie > n)
                    throw std::out_of_range("index out of range: particles [" + std::to_string(ib) + ", "
                                            + std::to_string(ie) + ")");
                DeviceGuard g(v->device);
                lam_cuda_check(lamk::nbody_update(v->img.hdr, f64, mode == LAM_NBODY_EXACT, particlePhys(v), n, ib, ie,
                                                  static_cast<cudaStream_t>(stream)),
                               "nbody_update");
                if(v->L->fac || v->L->heat)
                    lam_cuda_check(lamk::nbody_account(v->img.hdr, false, n, ib, ie, static_cast<cudaStream_t>(stream)),
                                   "nbody_account");
            });
    }

    int lam_nbody_update_multi(lam_view* v, const lam_view* const* jviews, const uint64_t* jbegin, const uint64_t* jend,
                               size_t nj, int mode, uint64_t ib, uint64_t ie, void* stream)
    {
        return guard2(
            [&]
            {
                const bool f64 = particleF64(v);
                const uint64_t n = v->L->map->elementCount();
                if(ib > ie || ie > n)
                    throw std::out_of_range("index out of range: particles [" + std::to_string(ib) + ", "
                                            + std::to_string(ie) + ")");
                if(nj == 0 || nj > 64 || !jviews || !jbegin || !jend)
                    throw std::invalid_argument("n-body j-sources: 1..64 views with ranges");
                if(v->L->fac || v->L->heat)
                    throw std::invalid_argument("instrumented views: use lam_nbody_update (single view)");
                bool phys = particlePhys(v);
                std::vector<const lamp_view*> hdr(nj);
                for(size_t k = 0; k < nj; ++k)
                {
                    const lam_view* j = jviews[k];
                    if(!(j->L->map->schema() == v->L->map->schema()) || !(j->L->map->extents() == v->L->map->extents()))
                        throw std::invalid_argument("incompatible views");
                    if(j->device != v->device)
                        throw std::invalid_argument("j-source views must live on the updating device (wrap peer memory)");
                    if(j->L->fac || j->L->heat)
                        throw std::invalid_argument("instrumented views: use lam_nbody_update (single view)");
                    if(jbegin[k] > jend[k] || jend[k] > n)
                        throw std::out_of_range("index out of range: j-source range");
                    phys = phys && particlePhys(j);
                    hdr[k] = j->img.hdr;
                }
                DeviceGuard g(v->device);
                lam_cuda_check(lamk::nbody_update_multi(v->img.hdr, f64, mode == LAM_NBODY_EXACT, phys, hdr.data(), jbegin,
                                                        jend, nj, ib, ie, static_cast<cudaStream_t>(stream)),
                               "nbody_update_multi");
            });
    }

    // CUDA IPC for the fused multi-GPU n-body step: a rank exports its blob allocations, the
    // others map them and wrap them as views (lam_view_wrap) on their own device
    int lam_ipc_get_handle(const void* device_ptr, void* handle_out)
    {
        return guard2(
            [&]
            {
                cudaIpcMemHandle_t h;
                lam_cuda_check(cudaIpcGetMemHandle(&h, const_cast<void*>(device_ptr)), "cudaIpcGetMemHandle");
                std::memcpy(handle_out, &h, sizeof(h));
            });
    }

    int lam_ipc_open(const void* handle, int device, void** device_ptr)
    {
        return guard2(
            [&]
            {
                DeviceGuard g(device);
                cudaIpcMemHandle_t h;
                std::memcpy(&h, handle, sizeof(h));
                lam_cuda_check(cudaIpcOpenMemHandle(device_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            });
    }

    int lam_ipc_close(void* device_ptr)
    {
        return guard2([&] { lam_cuda_check(cudaIpcCloseMemHandle(device_ptr), "cudaIpcCloseMemHandle"); });
    }

    int lam_nbody_step(lam_view* v, int mode, uint64_t ib, uint64_t ie, void* stream)
    {
        const int rc = lam_nbody_update(v, mode, ib, ie, stream);
        return rc != LAM_OK ? rc : lam_nbody_move(v, ib, ie, stream);
    }

    int lam_nbody_move(lam_view* v, uint64_t ib, uint64_t ie, void* stream)
    {
        return guard2(
            [&]
            {
                const bool f64 = particleF64(v);
                const uint64_t n = v->L->map->elementCount();
                if(ib > ie || ie > n)
                    throw std::out_of_range("index out of range: particles");
                DeviceGuard g(v->device);
                lam_cuda_check(lamk::nbody_move(v->img.hdr, f64, particlePhys(v), ib, ie, static_cast<cudaStream_t>(stream)),
                               "nbody_move");
                if(v->L->fac || v->L->heat)
                    lam_cuda_check(lamk::nbody_account(v->img.hdr, true, n, ib, ie, static_cast<cudaStream_t>(stream)),
                                   "nbody_account");
            });
    }

    int lam_nbody_pack_positions(const lam_view* v, uint64_t ib, uint64_t ie, int with_mass, void* out, void* stream)
    {
        return guard2(
            [&]
            {
                const bool f64 = particleF64(v);
                const uint64_t n = v->L->map->elementCount();
                if(ib > ie || ie > n)
                    throw std::out_of_range("index out of range: particles");
                if(!out && ie > ib)
                    throw std::invalid_argument("n-body pack: null output buffer");
                DeviceGuard g(v->device);
                lam_cuda_check(lamk::nbody_pack(v->img.hdr, f64, particlePhys(v), ib, ie, with_mass != 0, out,
                                                static_cast<cudaStream_t>(stream)),
                               "nbody_pack");
            });
    }

    int lam_nbody_checksum(const lam_view* v, double* out)
    {
        return guard2(
            [&]
            {
                const bool f64 = particleF64(v);
                DeviceGuard g(v->device);
                // checksumView takes no stream: order after all work on the device (non-blocking
                // streams included), then copy on the legacy stream and read back
                lam_cuda_check(cudaDeviceSynchronize(), "sync");
                const uint64_t n = v->L->map->elementCount();
                TempView tmp(*v, v->device);
                copyViews(*v, tmp.v, 0, n, nullptr);
                lam_cuda_check(cudaDeviceSynchronize(), "sync");
                const size_t T = f64 ? 8 : 4;
                std::vector<uint8_t> host(n * 7 * T);
                if(!host.empty())
                    lam_cuda_check(cudaMemcpy(host.data(), tmp.buf, host.size(), cudaMemcpyDeviceToHost), "d2h");
                // checksumView (runner.cpp:62-72): Σ x, y, z in double, index order
                double sum = 0;
                for(uint64_t i = 0; i < n; ++i)
                    for(int f = 0; f < 3; ++f)
                    {
                        if(f64)
                        {
                            double d;
                            std::memcpy(&d, &host[(i * 7 + f) * 8], 8);
                            sum += d;
                        }
                        else
                        {
                            float x;
                            std::memcpy(&x, &host[(i * 7 + f) * 4], 4);
                            sum += static_cast<double>(x);
                        }
                    }
                *out = sum;
            });
    }
}
