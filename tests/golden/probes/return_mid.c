#define N 8
double a[N];
int f(int c) {
    #pragma omp target teams distribute parallel for
    for (int k = 0; k < N; ++k) { a[k] = 1.0; }
    if (c > 0) {
        return 1;
    }
    a[0] = 2.0;
    #pragma omp target teams distribute parallel for
    for (int k = 0; k < N; ++k) { a[k] = a[k] + 1.0; }
    return 0;
}
