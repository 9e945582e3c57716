// Host cost of one lam_copy dispatch from C++ (no Python): small views, 2000 calls.
#include "lamina_b200.h"
#include <chrono>
#include <cstdio>
int main()
{
    const char* R = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}";
    const char* pairs[][2] = {{"aos-packed", "soa-mb"}, {"aos-packed", "bytesplit:soa-mb"}, {"soa-mb", "bitpack-float:8,10"},
                              {"aos-packed", "aos-packed"}};
    for(auto& pr : pairs)
    {
        lam_layout *a, *b;
        lam_view *va, *vb;
        lam_layout_create(R, "i32:[1024]", nullptr, 0, pr[0], 0, 0, &a);
        lam_layout_create(R, "i32:[1024]", nullptr, 0, pr[1], 0, 0, &b);
        lam_view_alloc(a, 0, nullptr, &va);
        lam_view_alloc(b, 0, nullptr, &vb);
        for(int k = 0; k < 50; ++k)
            lam_copy(va, vb, nullptr);
        lam_device_sync(0);
        auto t0 = std::chrono::steady_clock::now();
        for(int k = 0; k < 2000; ++k)
            lam_copy(va, vb, nullptr);
        auto t1 = std::chrono::steady_clock::now();
        lam_device_sync(0);
        std::printf("%s -> %s: %.2f us per lam_copy call\n", pr[0], pr[1],
                    std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000);
    }
}
