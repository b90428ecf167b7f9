// Dumps known-answer outputs of libcudacxx's cuda::std::philox4x32 (the C++26
// std::philox4x32) for tests/golden/philox_kat.json.  Built and run by
// tests/golden/make_golden.py in the build container only.
#include <cuda/std/__random/philox_engine.h>
#include <cstdio>
int main() {
    {
        cuda::std::philox4x32 e;  // default seed 20111115
        unsigned long long v = 0;
        for (int i = 0; i < 10000; ++i) v = e();
        std::printf("{\"default_10000th\": %llu, \"streams\": [", v);
    }
    const unsigned long long seeds[] = {0ull, 1ull, 20111115ull, 20260823ull, 0xffffffffull};
    for (int s = 0; s < 5; ++s) {
        cuda::std::philox4x32 e(seeds[s]);
        std::printf("%s{\"seed\": %llu, \"out\": [", s ? ", " : "", seeds[s]);
        for (int i = 0; i < 64; ++i) std::printf("%s%u", i ? ", " : "", (unsigned)e());
        std::printf("]}");
    }
    std::printf("]}\n");
    return 0;
}
