// TEST INFRASTRUCTURE: command-line front end of the reference n-body runner
// (proj/tools/nbody/runner.cpp) for golden-report generation.  The reference's own
// main.cpp needs CLI11 (absent); this one takes positional arguments:
//   ref_nbody <layout> <n> <steps> <f64 0|1> <seed> <trace 0|1> <heatmap granularity> <report dir>
// The runner's iostream/filesystem code runs in its own process: loaded into a Python
// process next to another libstdc++ it crashes, so the tests call this binary instead.
#include <cstdlib>

extern "C" int ref_nbody_trace(const char* layout, unsigned long long n, unsigned long long steps, int f64,
                               unsigned long long seed, int traceFields, unsigned long long heatGran,
                               const char* reportDir, const char* csvPath);

int main(int argc, char** argv)
{
    if(argc != 9)
        return 2;
    return ref_nbody_trace(argv[1], std::strtoull(argv[2], nullptr, 10), std::strtoull(argv[3], nullptr, 10),
                           std::atoi(argv[4]), std::strtoull(argv[5], nullptr, 10), std::atoi(argv[6]),
                           std::strtoull(argv[7], nullptr, 10), argv[8], nullptr);
}
