#define N 8
double a[N];
int main(int c) {
    #pragma omp target teams distribute parallel for
    for (int k = 0; k < N; ++k) { a[k] = 1.0; }
    if (c > 0) {
        a[1] = 5.0;
    } else {
        #pragma omp target teams distribute parallel for
        for (int k = 0; k < N; ++k) { a[k] = 2.0; }
    }
    double s = a[2];
    return (int) s;
}
