#define N 8
double a[N];
double b[N];
int main(int c) {
    #pragma omp target teams distribute parallel for
    for (int k = 0; k < N; ++k) { a[k] = 1.0; }
    if (c > 0) {
        if (c > 1) { b[0] = 1.0; }
        a[0] = 2.0;
    }
    double s = a[1];
    return (int) s;
}
