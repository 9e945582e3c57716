// Internal host structures behind the opaque C ABI handles.
#pragma once

#include "../../include/lamina_b200.h"
#include "host_layout.hpp"
#include "launch.h"

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

extern thread_local std::string g_lam_err;
void lam_cuda_check(cudaError_t e, const char* what);

namespace lamhost
{
    // one device allocation: lamp_view header + plan arrays + stream pointers + counters
    struct DeviceImage
    {
        int device = 0;
        void* mem = nullptr;
        void* heat = nullptr;
        size_t bytes = 0;
        size_t offRoots = 0, offNodes = 0, offStreams = 0, offPtrs = 0, offHeatOff = 0, offFac = 0;
        std::vector<uint8_t> host;
        const lamp_view* hdr = nullptr;
        unsigned long long* facDev = nullptr;

        DeviceImage() = default;
        DeviceImage(const DeviceImage&) = delete;
        DeviceImage& operator=(const DeviceImage&) = delete;
        ~DeviceImage();
        bool ownsHeat = true;
        // sharedHeat: counters owned by the caller (chunked pipelines share one heatmap)
        void build(const lamb::Lowered& L, int device, const std::vector<uint8_t*>& streamPtrs,
                   void* sharedHeat = nullptr);
        void setStreamPtrs(const std::vector<uint8_t*>& ptrs, cudaStream_t s);
        void release();
    };

    std::vector<uint8_t*> streamPtrsFor(const lamb::Lowered& L, const std::vector<void*>& blobs);

    struct DeviceGuard
    {
        int prev = -1;
        explicit DeviceGuard(int dev)
        {
            cudaGetDevice(&prev);
            if(prev != dev)
                lam_cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        }
        ~DeviceGuard()
        {
            int cur = -1;
            cudaGetDevice(&cur);
            if(prev >= 0 && cur != prev)
                cudaSetDevice(prev);
        }
    };

    template<typename T>
    struct DevBuf
    {
        T* p = nullptr;
        explicit DevBuf(size_t n)
        {
            if(n)
                lam_cuda_check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc(scratch)");
        }
        ~DevBuf()
        {
            if(p)
                cudaFree(p);
        }
        DevBuf(const DevBuf&) = delete;
        DevBuf& operator=(const DevBuf&) = delete;
    };
} // namespace lamhost

struct lam_layout
{
    std::shared_ptr<lamb::Lowered> L;
};

struct lam_view
{
    std::shared_ptr<lamb::Lowered> L;
    const lam_layout* layout = nullptr;
    int device = 0;
    bool owned = true;
    std::vector<void*> blobs;
    lamhost::DeviceImage img;
};

namespace lamhost
{
    // copyView over element range [begin, end) (view.cpp:168-189)
    void copyViews(const lam_view& src, lam_view& dst, uint64_t begin, uint64_t end, cudaStream_t s);
    void copyHost(const lam_layout& sl, const void* const* sb, const lam_layout& dl, void* const* db, int device,
                  uint64_t* srcCounters, uint64_t* dstCounters);

    // specialised tile engine; false when the pair is not tile-eligible (copy_tile_host.cpp)
    bool tileCopy(const lam_view& src, lam_view& dst, uint64_t begin, uint64_t end, cudaStream_t s);
    // same on raw images (used by the host pipeline's chunk views)
    bool tileCopyImages(const lamb::Lowered& SL, const DeviceImage& si, const lamb::Lowered& DL, DeviceImage& di,
                        uint64_t begin, uint64_t end, cudaStream_t s);
    // same with explicit (virtual) stream pointers, as chunk views use them
    bool tileCopyPtrs(const lamb::Lowered& SL, const DeviceImage& si, uint8_t* const* sptr, const lamb::Lowered& DL,
                      DeviceImage& di, uint8_t* const* dptr, uint64_t begin, uint64_t end, cudaStream_t s);
    bool tileEligible(const lamb::Lowered& SL, const lamb::Lowered& DL);

    // per-device chunked H2D -> copy -> D2H pipeline behind lam_copy_host (host_pipeline.cpp)
    class HostPipeline
    {
    public:
        static HostPipeline& get(int device);
        void run(const lam_layout& sl, const void* const* sb, const lam_layout& dl, void* const* db,
                 uint64_t* srcCounters, uint64_t* dstCounters);
        ~HostPipeline();

    private:
        explicit HostPipeline(int device);
        void ensure(size_t slotBytes);
        int device_;
        static constexpr int kSlots = 3;
        cudaStream_t h2d_ = nullptr, comp_ = nullptr, d2h_ = nullptr;
        cudaStream_t h2dB_ = nullptr, d2hB_ = nullptr; // second copy queue per direction
        cudaEvent_t evIn_[kSlots]{}, evDone_[kSlots]{}, evFree_[kSlots]{};
        cudaEvent_t evInB_[kSlots]{}, evFreeB_[kSlots]{};
        void* slot_[kSlots]{};
        size_t slotBytes_ = 0;
        void* pinnedPtrs_ = nullptr; // per slot stream-pointer tables (pinned)
        size_t pinnedBytes_ = 0;
        // per-slot chunk-view images, cached per (src, dst) layout pair
        struct Images
        {
            std::shared_ptr<lamb::Lowered> S, D;
            std::unique_ptr<DeviceImage> simg[kSlots], dimg[kSlots];
            void* sheat = nullptr;
            void* dheat = nullptr;
        };
        std::vector<std::unique_ptr<Images>> cache_;
        Images& images(const std::shared_ptr<lamb::Lowered>& S, const std::shared_ptr<lamb::Lowered>& D);
    };
} // namespace lamhost
