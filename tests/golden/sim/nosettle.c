#define N 8
double a[N];
double b[N];

int main() {
    for (int i = 0; i < 20000; i++) {
        #pragma omp target enter data map(to: a)
        a[0] = a[1] + 1.0;
        #pragma omp target update from(b)
        b[2] = a[3];
    }
    for (int j = 0; j < 30; j++) {
        #pragma omp target teams distribute parallel for
        for (int k = 0; k < N; k++) {
            b[k] = a[k] * 2.0;
        }
    }
    return 0;
}
