#define N 8
double a[N];
int main(int c) {
    #pragma omp target teams distribute parallel for
    for (int k = 0; k < N; ++k) { a[k] = 1.0; }
    switch (c) {
    case 1:
        a[3] = a[2];
    case 2:
        a[4] = 1.0;
        break;
    }
    return (int) a[0];
}
