// Host cost of a kernel launch as a function of the kernel-parameter size
// (diagnostic for the exchange kernels' ~3.4 KB ExchParams).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
struct P { unsigned char b[N]; };

template <int N>
__global__ void k(const __grid_constant__ P<N> p) {
    if (threadIdx.x == 0 && p.b[0] == 255 && p.b[N - 1] == 255) printf("x");
}

template <int N>
double time_launch(int reps, bool coop) {
    P<N> p{};
    void *args[] = {&p};
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int i = 0; i < 100; ++i) cudaLaunchKernel((const void *)k<N>, dim3(4), dim3(256), args, 0, s);
    cudaStreamSynchronize(s);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) {
        if (coop)
            cudaLaunchCooperativeKernel((const void *)k<N>, dim3(4), dim3(256), args, 0, s);
        else
            cudaLaunchKernel((const void *)k<N>, dim3(4), dim3(256), args, 0, s);
    }
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t2 = std::chrono::steady_clock::now();
    cudaStreamDestroy(s);
    printf("params %5d B %s: %.2f us/launch issue, %.2f us/launch incl. drain\n", N, coop ? "coop " : "plain",
           std::chrono::duration<double, std::micro>(t1 - t0).count() / reps,
           std::chrono::duration<double, std::micro>(t2 - t0).count() / reps);
    return 0;
}

int main() {
    for (int coop = 0; coop < 2; ++coop) {
        time_launch<64>(5000, coop);
        time_launch<512>(5000, coop);
        time_launch<1024>(5000, coop);
        time_launch<2048>(5000, coop);
        time_launch<3584>(5000, coop);
        time_launch<8192>(5000, coop);
    }
    return 0;
}
